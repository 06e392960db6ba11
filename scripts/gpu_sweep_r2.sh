# Round-2 config sweep on the final kernels: bench line per BASELINE config, SURVEY 8(f) rows
# (construction / add / truncate), variants, approximate, bs 16 layouts. Usage: bash scripts/gpu_sweep_r2.sh TAG
TAG=${1:-R2s}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
for C in C1 C2-16384 C2-32768 C2-65536 C2-131072 C3 C4 C5-32 C5-64 C5-128; do
  timeout 900 python bench.py --config $C --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_${TAG}_$C.json.log 2>&1; echo "bench $C rc=$?"
  tail -1 gpurun_out/bench_${TAG}_$C.json.log > gpurun_out/bench_${TAG}_$C.json
done
timeout 600 python scripts/fnext_probe.py --out gpurun_out/fnext_$TAG.json > gpurun_out/fnext_$TAG.log 2>&1; echo "fnext rc=$?"
timeout 600 python scripts/variants_probe.py > gpurun_out/variants_$TAG.txt 2>&1; echo "variants rc=$?"
timeout 300 python scripts/approx_probe.py --out gpurun_out/approx_$TAG.json > gpurun_out/approx_$TAG.log 2>&1; echo "approx rc=$?"
timeout 300 python scripts/layout_phase_probe.py > gpurun_out/layout_$TAG.txt 2>&1; echo "layout rc=$?"
