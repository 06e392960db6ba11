timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "rank_ordering or symbolic" 2>&1 | tail -2
for c in C2-16384 C3 C2-65536 C2-131072; do for r in 1 0 1 0; do
  QM_RANK_ORDER=$r timeout 300 python bench.py --config $c --no-e2e --no-cpu --steps 30 2>/dev/null | python -c "
import sys, json
d = json.loads(sys.stdin.readlines()[-1]); print('$c rank=$r', d['ms_per_step'], d['phases_ms'])"
done; done
