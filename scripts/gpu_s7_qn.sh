for q in 1 0; do
TAG=q32_$q
K=k_numeric_quad32; [ $q = 0 ] && K=k_numeric_tma
QM_QUAD32=$q timeout 600 ncu --set full --clock-control none --import-source on -k regex:$K -s 1 -c 1 -o gpurun_out/prof_$TAG python scripts/bs32_probe.py > gpurun_out/ncu_$TAG.log 2>&1; echo "ncu rc=$?"
ncu -i gpurun_out/prof_$TAG.ncu-rep --page raw --csv > gpurun_out/ncu_raw_$TAG.csv 2>/dev/null
ncu -i gpurun_out/prof_$TAG.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu_src_$TAG.csv 2>/dev/null
done
