# Round-2 evidence run on one B200: C5-64 e2e timeline, the bench's ncu launch list (C5-64),
# a targeted ncu capture of k_numeric_tma on C5-64 (application replay: the kernel writes 35 GB,
# too much for kernel-replay save/restore), and the real reference timed on the host.
# Usage: bash scripts/gpu_r2_profile.sh TAG
TAG=${1:-R2}
mkdir -p gpurun_out
timeout 900 python scripts/e2e_c5_probe.py > gpurun_out/e2e_c5_$TAG.log 2>&1; echo "e2e probe rc=$?"
CMD="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_C5-64_$TAG.csv $CMD > gpurun_out/ncu_launches_$TAG.log 2>&1; echo "ncu launches rc=$?"
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_tensor_subpipe_dmma.sum,lts__t_sector_hit_rate.pct,sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread,launch__grid_size,sm__cycles_elapsed.avg.per_second
timeout 1500 ncu --replay-mode application --metrics $M --clock-control none -k regex:k_numeric_tma -c 1 -o gpurun_out/prof_c5_$TAG python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu > gpurun_out/ncu_c5_$TAG.log 2>&1; echo "ncu C5 rc=$?"
ncu -i gpurun_out/prof_c5_$TAG.ncu-rep --page raw --csv > gpurun_out/prof_c5_$TAG.csv 2>/dev/null
timeout 1200 python scripts/reference_cpu_timing.py gpurun_out/reference_quadmat_$TAG.json > gpurun_out/refcpu_$TAG.log 2>&1; echo "reference cpu rc=$?"
