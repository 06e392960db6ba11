timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "quad or adversarial or grouped" 2>&1 | tail -2
for i in 1 2; do timeout 600 python bench.py --config C5-32 --no-e2e --no-cpu --steps 5 2>/dev/null | python -c "
import sys, json
d = json.loads(sys.stdin.readlines()[-1]); print('C5-32', d['ms_per_step'], d['phases_ms'], d['roofline']['kernel'], d['roofline']['frac'])"; done
QM_QUAD32=1 timeout 300 python scripts/layout_phase_probe.py 2>&1 | grep "bs 32 tma"
