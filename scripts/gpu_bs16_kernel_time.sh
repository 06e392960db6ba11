# bs 16 kernel-only time (ncu gpu__time_duration of k_numeric_group16) for experimental builds.
for v in $1; do
  QM_LIB_PATH=exp_lib/libqmb200_$v.so timeout 600 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:k_numeric_group16 -s 3 -c 1 --csv python scripts/bs16_probe.py 2>/dev/null | grep -E "gpu__time|dmma" | sed "s/^/$v: /" | cut -c1-200
done
