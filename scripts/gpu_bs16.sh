# bs 16 grouped kernel: tests, per-layout phase times, ncu full capture of k_numeric_group16.
TAG=${1:-r}
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -q -k "bs16 or special_values" > gpurun_out/t_bs16_$TAG.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/t_bs16_$TAG.log
timeout 300 python scripts/layout_phase_probe.py > gpurun_out/layout_$TAG.log 2>&1; echo "probe rc=$?"; head -3 gpurun_out/layout_$TAG.log
timeout 300 python scripts/bs16_probe.py > /dev/null 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_numeric_group16 -s 1 -c 1 -o gpurun_out/prof_bs16_$TAG python scripts/bs16_probe.py > gpurun_out/ncu_bs16_$TAG.log 2>&1; echo "ncu rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bs16_$TAG.csv python scripts/bs16_probe.py > /dev/null 2>&1; echo "launches rc=$?"
