# Distributed structure cache: multirank / partition GPU tests, torchrun path check, projection.
timeout 1200 python -m pytest tests/test_gpu_multirank.py tests/test_gpu_partition.py -q -x 2>&1 | tail -2
bash scripts/gpu_torchrun_check.sh 2>&1 | grep -E "rc="
timeout 1500 python scripts/scaling_projection.py --out gpurun_out/proj_Z2.json > gpurun_out/proj_Z2.log 2>&1; echo "proj rc=$?"; tail -12 gpurun_out/proj_Z2.log
