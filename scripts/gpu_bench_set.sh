# bench lines for a set of configs (no e2e / cpu legs). Usage: bash scripts/gpu_bench_set.sh TAG STEPS CONFIG...
TAG=$1; STEPS=$2; shift 2
mkdir -p gpurun_out
for C in "$@"; do
  timeout 600 python bench.py --config $C --steps $STEPS --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_${TAG}_${C}.log 2>&1; echo "bench $C rc=$?"
  python -c "
import json
l=json.loads(open('gpurun_out/bench_${TAG}_${C}.log').read().strip().splitlines()[-1])
print(l['config']['workload'], l['value'], l['ms_per_step'], l['phases_ms'], l['roofline']['achieved'], l['roofline']['frac'], l['clocks'])" 2>&1 | tail -2
done
