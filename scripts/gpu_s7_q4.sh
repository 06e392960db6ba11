timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "quad" 2>&1 | tail -2
for q in 1 0; do
  QM_QUAD32=$q timeout 600 python bench.py --config C5-32 --no-e2e --no-cpu --steps 5 2>/dev/null | python -c "
import sys, json
d = json.loads(sys.stdin.readlines()[-1]); print('C5-32 quad=$q', d['ms_per_step'], d['phases_ms'], d['roofline']['achieved'], d['roofline']['frac'])"
done
QM_QUAD32=1 QM_QUAD32_VARIANT=deep timeout 600 python bench.py --config C5-32 --no-e2e --no-cpu --steps 5 2>/dev/null | python -c "
import sys, json
d = json.loads(sys.stdin.readlines()[-1]); print('C5-32 quad deep', d['ms_per_step'], d['phases_ms'], d['roofline']['achieved'], d['roofline']['frac'])"
for q in 1 0; do QM_QUAD32=$q timeout 300 python scripts/layout_phase_probe.py 2>&1 | grep "bs 32 tma" | sed "s/^/quad=$q /"; done
