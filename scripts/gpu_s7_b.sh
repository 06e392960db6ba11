# Inline merge of the bs 16 grouped kernel (A/B against the merge pass) + medium single-CTA sort A/B.
timeout 900 python -m pytest tests -m gpu -q -x -k "bs16 or group or layout or default" 2>&1 | tail -3
for m in inline kernel inline kernel; do QM_G16_MERGE=$m timeout 300 python scripts/bs16_size_probe.py 32768 262144 2>&1 | grep "^n " | sed "s/^/$m: /"; done
for c in C1 C2-16384 C2-32768; do for ss in 1 0 1 0; do
  QM_SMALL_SORT=$ss timeout 300 python bench.py --config $c --no-e2e --no-cpu --steps 30 2>/dev/null | python -c "
import sys, json
d = json.loads(sys.stdin.readlines()[-1]); print('$c small_sort=$ss', d['ms_per_step'], d['phases_ms'])"
done; done
timeout 900 python -m pytest tests -m gpu -q -x -k "C2 or symbolic or baseline" 2>&1 | tail -3
