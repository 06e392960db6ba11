# Full GPU suite on the new bs 16 kernel + its ncu capture (source counters) + sanitizer pass of the bs 16 tests.
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_s7f.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu_s7f.log
bash scripts/gpu_bs16_ncu.sh s7f
timeout 900 compute-sanitizer --tool memcheck python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "bs16_inline" > gpurun_out/sanitizer_s7f.log 2>&1; echo "memcheck rc=$?"; tail -4 gpurun_out/sanitizer_s7f.log
timeout 900 compute-sanitizer --tool racecheck python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "bs16_inline and 1000" > gpurun_out/racecheck_s7f.log 2>&1; echo "racecheck rc=$?"; tail -4 gpurun_out/racecheck_s7f.log
