timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "quad" 2>&1 | tail -3
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -3
