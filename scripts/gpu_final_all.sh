# Final round-2 evidence run: GPU tests, smoke, default bench + reference arm, config sweep,
# SURVEY 8(f) rows, scaling projection. Usage: bash scripts/gpu_final_all.sh TAG
TAG=${1:-Z}
bash scripts/gpu_head_check.sh $TAG
bash scripts/gpu_sweep_r2.sh R2s
timeout 1500 python scripts/scaling_projection.py --out gpurun_out/proj_$TAG.json > gpurun_out/proj_$TAG.log 2>&1; echo "proj rc=$?"; tail -12 gpurun_out/proj_$TAG.log
