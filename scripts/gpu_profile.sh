# Round profile: default bench line (e2e + cpu baseline), reference arm, config sweep, ncu evidence.
TAG=${1:-r}
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_default_$TAG.log 2>&1; echo "bench default rc=$?"; tail -1 gpurun_out/bench_default_$TAG.log | cut -c1-300
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_reference_$TAG.log 2>&1; echo "bench reference rc=$?"; tail -1 gpurun_out/bench_reference_$TAG.log | cut -c1-200
for C in C1 C2-16384 C2-32768 C2-65536 C2-131072 C3 C4 C5-32 C5-64 C5-128; do
  timeout 600 python bench.py --config $C --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_${TAG}_$C.log 2>&1; echo "bench $C rc=$?"
done
CMD="python bench.py --config C2-131072 --steps 2 --warmup 1 --no-e2e --no-cpu"
$CMD > gpurun_out/ncu_plain_$TAG.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_launch_$TAG.log 2>&1; echo "ncu launches rc=$?"
$CMD > gpurun_out/ncu_plain2_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_numeric_tma -s 1 -c 1 -o gpurun_out/prof_numeric_$TAG $CMD > gpurun_out/ncu_full_$TAG.log 2>&1; echo "ncu full rc=$?"
