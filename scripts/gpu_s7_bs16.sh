# bs 16: size dependence of the default build, then A/B of experimental builds (layout probe bs-16 row + kernel-only time).
python scripts/bs16_size_probe.py 32768 131072 262144 2>&1 | grep "^n "
bash scripts/gpu_bs16_ab.sh "$1"
for v in $1; do QM_LIB_PATH=exp_lib/libqmb200_$v.so timeout 300 python scripts/bs16_size_probe.py 262144 2>&1 | grep "^n " | sed "s/^/$v: /"; done
timeout 600 python -m pytest tests -m gpu -q -k "bs16 or group" 2>&1 | tail -2
for v in $1; do QM_LIB_PATH=exp_lib/libqmb200_$v.so timeout 600 python -m pytest tests -m gpu -q -k "bs16 or group" 2>&1 | tail -1 | sed "s/^/$v: /"; done
