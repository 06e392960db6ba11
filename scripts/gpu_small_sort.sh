# Single-CTA C-key sort for small products: symbolic / partition / parity tests, then A/B.
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_partition.py -q -x 2>&1 | tail -2
for c in C1 C2-16384 C4; do for ss in 1 0; do
  QM_SMALL_SORT=$ss timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu 2>/dev/null | tail -1 | python -c "
import json,sys; l=json.loads(sys.stdin.read()); print('$c small_sort=$ss step', l['ms_per_step'], l['phases_ms'])"
done; done
