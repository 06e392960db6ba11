# bs 16: compile-time specialised partial stages (this build) on top of the inline merge.
timeout 900 python -m pytest tests -m gpu -q -x -k "bs16 or group or layout or default" 2>&1 | tail -3
for m in inline inline; do QM_G16_MERGE=$m timeout 300 python scripts/bs16_size_probe.py 32768 262144 2>&1 | grep "^n " | sed "s/^/$m: /"; done
timeout 300 python scripts/layout_phase_probe.py 2>&1 | grep "bs 16"
timeout 300 python scripts/kernel_families_probe.py 2>&1 | tail -12
