TAG=${1:-r02}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_gpu_$TAG.log
for C in C2-131072 C5-64 C5-128 C5-32 C3 C4; do
  for IMPL in tma cpasync; do
    QM_NUMERIC=$IMPL timeout 600 python bench.py --config $C --steps 5 --warmup 2 --no-e2e --no-cpu > gpurun_out/bench_${TAG}_${C}_$IMPL.log 2>&1; echo "bench $C $IMPL rc=$?"
    python -c "
import json,sys
l=json.loads(open('gpurun_out/bench_${TAG}_${C}_$IMPL.log').read().strip().splitlines()[-1])
print(l['config']['workload'], '$IMPL', l['value'], l['ms_per_step'], l['phases_ms'], l['roofline']['achieved'], l['roofline']['frac'], l['clocks'])" 2>&1 | tail -2
  done
done
