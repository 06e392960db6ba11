# bs 16 variants (exp_lib builds): numeric phase of the layout probe's bs-16 row.
for v in $1; do for rep in 1 2; do
  QM_LIB_PATH=exp_lib/libqmb200_$v.so timeout 300 python scripts/layout_phase_probe.py 2>&1 | grep "bs 16 tma  " | sed "s/^/$v rep$rep: /"
done; done
