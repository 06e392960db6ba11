# bs 16 grouped kernel: one ncu --set full capture with source counters (stall reasons per SASS line).
TAG=${1:-b16}
mkdir -p gpurun_out
timeout 300 python scripts/bs16_probe.py > /dev/null 2>&1; echo "probe rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_numeric_group16 -s 1 -c 1 -o gpurun_out/prof_$TAG python scripts/bs16_probe.py > gpurun_out/ncu_$TAG.log 2>&1; echo "ncu rc=$?"
ncu -i gpurun_out/prof_$TAG.ncu-rep --page raw --csv > gpurun_out/ncu_raw_$TAG.csv 2>/dev/null
ncu -i gpurun_out/prof_$TAG.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu_src_$TAG.csv 2>/dev/null
timeout 300 python scripts/layout_phase_probe.py 2>&1 | head -4
