timeout 900 python -m pytest tests -m gpu -q -x -k "bs16 or group or layout or default or families" 2>&1 | tail -2
for i in 1 2; do timeout 300 python scripts/bs16_size_probe.py 32768 262144 2>&1 | grep "^n "; done
timeout 300 python scripts/layout_phase_probe.py 2>&1 | grep "bs 16"
timeout 300 python scripts/kernel_families_probe.py 2>&1 | tail -7
