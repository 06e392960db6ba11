# Small-config evidence: symbolic probe, C1/C3 launch lists, ncu full of the numeric kernel.
# Usage: bash scripts/gpu_small_profile.sh TAG
TAG=${1:-r}
mkdir -p gpurun_out
timeout 300 python scripts/symbolic_probe.py C1 C3 C2-16384 > gpurun_out/symprobe_$TAG.log 2>&1; echo "symprobe rc=$?"
for C in C1 C3; do
  CMD="python bench.py --config $C --steps 3 --warmup 3 --no-e2e --no-cpu"
  timeout 300 $CMD > gpurun_out/plain_${TAG}_$C.log 2>&1; echo "plain $C rc=$?"
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}_$C.csv $CMD > /dev/null 2>&1; echo "launches $C rc=$?"
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_numeric_tma -s 2 -c 1 -o gpurun_out/prof_${TAG}_$C $CMD > gpurun_out/ncu_full_${TAG}_$C.log 2>&1; echo "ncu $C rc=$?"
done
