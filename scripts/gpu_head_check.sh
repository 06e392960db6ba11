# Full HEAD check on one B200: GPU tests, smoke, default bench line (C5-64 with e2e + cpu_baseline),
# and the reference arm. Usage: bash scripts/gpu_head_check.sh TAG
TAG=${1:-h}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_gpu_$TAG.log
timeout 300 python __graft_entry__.py --smoke > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke_$TAG.log
timeout 900 python bench.py > gpurun_out/bench_$TAG.log 2>&1; echo "bench rc=$?"; tail -2 gpurun_out/bench_$TAG.log
timeout 600 python bench.py --impl reference > gpurun_out/benchref_$TAG.log 2>&1; echo "benchref rc=$?"; tail -2 gpurun_out/benchref_$TAG.log
