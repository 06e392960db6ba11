timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -3
python scripts/bs16_random_probe.py 2>&1 | grep -v Warn | tail -8
timeout 600 python /tmp/none 2>/dev/null
python scripts/bs16_size_probe.py 32768 262144 2>&1 | grep "^n "
