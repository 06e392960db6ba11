# ncu evidence for the bs 32 quad kernel on C5-32: DRAM traffic + DMMA pipe (application replay: the
# kernel writes 35 GB), plus a --set full capture with source counters on the small banded probe.
TAG=${1:-Q}
mkdir -p gpurun_out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_tensor_subpipe_dmma.sum,lts__t_sector_hit_rate.pct,launch__registers_per_thread,launch__grid_size,sm__cycles_elapsed.avg.per_second
timeout 1500 ncu --replay-mode application --metrics $M --clock-control none -k regex:k_numeric_quad32 -c 1 --csv python bench.py --config C5-32 --steps 1 --warmup 0 --no-e2e --no-cpu > gpurun_out/ncu_C5-32_$TAG.csv 2> gpurun_out/ncu_C5-32_$TAG.err; echo "ncu C5-32 rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_numeric_quad32 -s 1 -c 1 -o gpurun_out/prof_quad_$TAG python scripts/bs32_probe.py > gpurun_out/ncu_quad_$TAG.log 2>&1; echo "ncu full rc=$?"
ncu -i gpurun_out/prof_quad_$TAG.ncu-rep --page raw --csv > gpurun_out/ncu_raw_quad_$TAG.csv 2>/dev/null
ncu -i gpurun_out/prof_quad_$TAG.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu_src_quad_$TAG.csv 2>/dev/null
python -c "import bench; print('quad kernel source', bench.kernel_source_sha('k_numeric_quad32'))"
