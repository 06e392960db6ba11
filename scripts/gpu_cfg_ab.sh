# A/B of bench configs under two env settings. Usage: bash scripts/gpu_cfg_ab.sh TAG "ENV_A" "ENV_B" CONFIG...
TAG=$1; EA=$2; EB=$3; shift 3
mkdir -p gpurun_out
for C in "$@"; do
  for E in "$EA" "$EB"; do
    env $E timeout 300 python bench.py --config $C --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/ab_${TAG}.log 2>&1 || echo "bench $C $E failed"
    tail -1 gpurun_out/ab_${TAG}.log | python -c "import json,sys; l=json.loads(sys.stdin.read()); print('$C', '$E', l['ms_per_step'], l['phases_ms'], l['roofline']['achieved'], l['roofline']['frac'], l['clocks']['sm_mhz'])"
  done
done
