# Round-2 state check: bench lines of the configs the open items are about, approximate vs regular
# on C4, bs16 phase times and the scaling projection. Usage: bash scripts/gpu_state_r2.sh TAG
TAG=${1:-s}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
bash scripts/gpu_bench_set.sh $TAG 10 C3 C4 C2-16384 C1
timeout 300 python scripts/approx_probe.py --out gpurun_out/approx_$TAG.json > gpurun_out/approx_$TAG.log 2>&1; echo "approx rc=$?"; cat gpurun_out/approx_$TAG.log | tail -5
timeout 300 python scripts/layout_phase_probe.py > gpurun_out/layout_$TAG.log 2>&1; echo "layout rc=$?"; head -12 gpurun_out/layout_$TAG.log
timeout 900 python scripts/scaling_projection.py --out gpurun_out/proj_$TAG.json > gpurun_out/proj_$TAG.log 2>&1; echo "proj rc=$?"; tail -14 gpurun_out/proj_$TAG.log
