# C4 multi-GPU work: partition / staged / multirank tests, staged-step timeline, projection.
TAG=${1:-c}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_partition.py tests/test_gpu_multirank.py -x -q > gpurun_out/t_part_$TAG.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/t_part_$TAG.log
timeout 300 python scripts/staged_probe.py C4 8 4 > gpurun_out/staged_probe_$TAG.log 2>&1; echo "probe rc=$?"; grep -E "^\{|host ms|k_halo|k_numeric|k_stage|span|step ms" gpurun_out/staged_probe_$TAG.log
timeout 900 python scripts/scaling_projection.py --configs ${CONFIGS:-C4} --out gpurun_out/proj_$TAG.json > gpurun_out/proj_$TAG.log 2>&1; echo "proj rc=$?"; tail -14 gpurun_out/proj_$TAG.log
