# Perf sweep + ncu evidence for the numeric kernel. Usage: bash scripts/gpu_perf.sh <tag>
TAG=${1:-r01}
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu_$TAG.log
for C in C1 C3 C4 C2-16384 C2-131072 C5-64 C5-128 C5-32; do
  timeout 600 python bench.py --config $C --steps 5 --warmup 2 --no-e2e --no-cpu > gpurun_out/bench_${TAG}_$C.log 2>&1; echo "bench $C rc=$?"; tail -1 gpurun_out/bench_${TAG}_$C.log | cut -c1-400
done
CMD="python bench.py --config C2-131072 --steps 2 --warmup 1 --no-e2e --no-cpu"
$CMD > gpurun_out/ncu_plain_$TAG.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_launch_$TAG.log 2>&1; echo "ncu launches rc=$?"
$CMD > gpurun_out/ncu_plain2_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_numeric_dmma -s 1 -c 1 -o gpurun_out/prof_numeric_$TAG $CMD > gpurun_out/ncu_full_$TAG.log 2>&1; echo "ncu full rc=$?"
tail -3 gpurun_out/ncu_full_$TAG.log
