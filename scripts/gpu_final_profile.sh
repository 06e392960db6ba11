# Final round profile: tests, smoke, default/reference lines, config sweep, ncu (C2-131072 launch
# list + full capture), plus full captures of the masked (C4) and transposed-reference
# (symmetric_square) numeric kernels, 8(f) rows and variants. Usage: bash scripts/gpu_final_profile.sh TAG
TAG=${1:-r}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/t_$TAG.log 2>&1; echo "pytest rc=$?"; grep -E "FAILED|passed|failed" gpurun_out/t_$TAG.log | tail -3
timeout 300 python __graft_entry__.py --smoke > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke_$TAG.log
bash scripts/gpu_profile.sh $TAG
timeout 300 python scripts/variants_probe.py > gpurun_out/variants_$TAG.log 2>&1; echo "variants rc=$?"
timeout 600 python scripts/fnext_probe.py --out gpurun_out/fnext_$TAG.json > gpurun_out/fnext_$TAG.log 2>&1; echo "fnext rc=$?"
CMD="python bench.py --config C4 --steps 2 --warmup 1 --no-e2e --no-cpu"
$CMD > /dev/null 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_numeric_tma -s 1 -c 1 -o gpurun_out/prof_c4_$TAG $CMD > gpurun_out/ncu_c4_$TAG.log 2>&1; echo "ncu C4 rc=$?"
timeout 600 ncu --set full --clock-control none --kernel-name-base mangled -k regex:"k_numeric_tma.*Lb1E" -c 1 -o gpurun_out/prof_symsq_$TAG python scripts/variants_probe.py > gpurun_out/ncu_symsq_$TAG.log 2>&1; echo "ncu symsq rc=$?"
