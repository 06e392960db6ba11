# tests + a few bench configs. Usage: bash scripts/gpu_quick.sh TAG CONFIG...
TAG=$1; shift
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/pytest_gpu_$TAG.log
for C in "$@"; do
  timeout 600 python bench.py --config $C --steps 5 --warmup 2 --no-e2e --no-cpu > gpurun_out/bench_${TAG}_${C}.log 2>&1; echo "bench $C rc=$?"
  python -c "
import json
l=json.loads(open('gpurun_out/bench_${TAG}_${C}.log').read().strip().splitlines()[-1])
print(l['config']['workload'], l['value'], l['ms_per_step'], l['phases_ms'], l['roofline']['achieved'], l['roofline']['frac'], l['clocks'])" 2>&1 | tail -2
done
