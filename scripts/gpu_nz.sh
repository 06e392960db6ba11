# Exact-zero flag from the sum of squares: parity, then A/B against the per-value compare.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/t_parity_nz.log 2>&1; echo "parity rc=$?"; tail -1 gpurun_out/t_parity_nz.log
bash scripts/gpu_lib_ab.sh "base nzfp" "C3 C2-16384 C4 C2-131072" nz2 2
