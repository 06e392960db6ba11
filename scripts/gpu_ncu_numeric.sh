# ncu --set full capture of the numeric kernel for one config. Usage: bash scripts/gpu_ncu_numeric.sh TAG CONFIG
TAG=$1; C=${2:-C2-131072}
mkdir -p gpurun_out
CMD="python bench.py --config $C --steps 2 --warmup 1 --no-e2e --no-cpu"
$CMD > gpurun_out/ncu_plain_${TAG}_$C.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_numeric_tma -s 1 -c 1 -o gpurun_out/prof_${TAG}_$C $CMD > gpurun_out/ncu_full_${TAG}_$C.log 2>&1; echo "ncu rc=$?"
