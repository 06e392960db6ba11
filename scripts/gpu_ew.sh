# Epilogue-warp variants: parity of bs-64 paths under each, then A/B against the in-warp epilogue.
TAG=${1:-ew}
mkdir -p gpurun_out
for ew in 1 2; do QM_EPILOGUE_WARP=$ew timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/t_parity_${TAG}_$ew.log 2>&1; echo "parity ew=$ew rc=$?"; tail -1 gpurun_out/t_parity_${TAG}_$ew.log; done
for c in C3 C2-16384 C1; do for ew in 2 0 1; do
  QM_EPILOGUE_WARP=$ew timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu 2>/dev/null | tail -1 | python -c "
import json,sys; l=json.loads(sys.stdin.read()); print('$c ew=$ew', l['phases_ms'], round(l['roofline']['achieved'],2), round(l['roofline']['frac'],4))"
done; done
