mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "numeric_kernel or both_numeric" > gpurun_out/pytest_bs16.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/pytest_bs16.log
timeout 300 python scripts/default_layout_probe.py 2>&1 | tail -4
QM_NUMERIC=cpasync timeout 300 python scripts/default_layout_probe.py 2>&1 | tail -4
