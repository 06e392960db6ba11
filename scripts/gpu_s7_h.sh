timeout 900 python -m pytest tests -m gpu -q -x -k "single_cta_sort or symbolic or row_index" 2>&1 | tail -2
for c in C2-16384 C1; do for ss in 1 0 1 0; do
  QM_SMALL_SORT=$ss timeout 300 python bench.py --config $c --no-e2e --no-cpu --steps 30 2>/dev/null | python -c "
import sys, json
d = json.loads(sys.stdin.readlines()[-1]); print('$c small_sort=$ss', d['ms_per_step'], d['phases_ms'])"
done; done
