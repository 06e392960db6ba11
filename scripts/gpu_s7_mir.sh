for v in "" exp_lib/libqmb200_g16mir.so "" exp_lib/libqmb200_g16mir.so; do QM_LIB_PATH=$v timeout 300 python scripts/bs16_size_probe.py 32768 262144 2>&1 | grep "^n " | sed "s|^|[$v] |"; done
QM_LIB_PATH=exp_lib/libqmb200_g16mir.so timeout 900 python -m pytest tests -m gpu -q -x -k "bs16 or group or adversarial or families" 2>&1 | tail -2
