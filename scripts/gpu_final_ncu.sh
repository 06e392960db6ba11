# Final ncu evidence on the current kernel sources: the bench's launch list (C5-64), DRAM traffic
# + DMMA pipe of k_numeric_tma per workload (application replay for C5-64, whose kernel writes
# 35 GB; kernel replay for the others). Usage: bash scripts/gpu_final_ncu.sh TAG
TAG=${1:-F}
mkdir -p gpurun_out
python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > gpurun_out/plain_$TAG.log 2>&1; echo "plain rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_C5-64_$TAG.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_launches_$TAG.log 2>&1; echo "launches rc=$?"
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_tensor_subpipe_dmma.sum,lts__t_sector_hit_rate.pct,launch__registers_per_thread,launch__grid_size,sm__cycles_elapsed.avg.per_second
timeout 1500 ncu --replay-mode application --metrics $M --clock-control none -k regex:k_numeric_tma -c 1 --csv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu > gpurun_out/ncu_C5-64_$TAG.csv 2> gpurun_out/ncu_C5-64_$TAG.err; echo "ncu C5-64 rc=$?"
for C in C2-131072 C3 C4; do
  timeout 900 ncu --metrics $M --clock-control none -k regex:k_numeric_tma -s 1 -c 1 --csv python bench.py --config $C --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_${C}_$TAG.csv 2> gpurun_out/ncu_${C}_$TAG.err; echo "ncu $C rc=$?"
done
python -c "import bench; print('kernel source', bench.kernel_source_sha())"
