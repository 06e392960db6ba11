timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "rank_ordering or symbolic or single_cta or row_index" 2>&1 | tail -2
for c in C1 C2-16384 C2-32768 C3 C4 C2-131072; do for r in 1 0 1 0; do
  QM_RANK_ORDER=$r timeout 300 python bench.py --config $c --no-e2e --no-cpu --steps 30 2>/dev/null | python -c "
import sys, json
d = json.loads(sys.stdin.readlines()[-1]); print('$c rank=$r', d['ms_per_step'], d['phases_ms'])"
done; done
QM_SMALL_SORT=0 timeout 300 python bench.py --config C1 --no-e2e --no-cpu --steps 30 2>/dev/null | python -c "
import sys, json
d = json.loads(sys.stdin.readlines()[-1]); print('C1 rank forced', d['ms_per_step'], d['phases_ms'])"
