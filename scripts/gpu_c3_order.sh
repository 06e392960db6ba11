# C3 claim-order check: GPU tests, C3 bench in k order (default) and key order, ncu DRAM bytes.
TAG=${1:-r}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu_$TAG.log
for O in k key; do
  QM_UNIT_ORDER=$O timeout 300 python bench.py --config C3 --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_${TAG}_C3_$O.log 2>&1; echo "bench $O rc=$?"
  tail -1 gpurun_out/bench_${TAG}_C3_$O.log | python -c "import json,sys; l=json.loads(sys.stdin.read()); print(l['ms_per_step'], l['phases_ms'], l['roofline']['achieved'], l['roofline']['frac'])"
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_numeric_tma -s 2 -c 1 -o gpurun_out/prof_${TAG}_C3 python bench.py --config C3 --steps 2 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_${TAG}_C3.log 2>&1; echo "ncu rc=$?"
