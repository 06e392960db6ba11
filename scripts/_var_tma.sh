for V in "0 0" "1 0" "0 1" "1 1"; do
  set -- $V
  QM_NVCC_EXTRA="-DQM_EXP_PRELOAD=$1 -DQM_EXP_EPI=$2" python -c "from paper_2011_11762_b200 import _build; _build.build(force=True, verbose=False)" > /dev/null 2>&1 || echo "build fail $V"
  for C in C3 C2-131072 C3; do
    QM_UNIT_ORDER=key timeout 300 python bench.py --config $C --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/v.log 2>&1
    tail -1 gpurun_out/v.log | python -c "import json,sys; l=json.loads(sys.stdin.read()); print('preload=$1 epi=$2', '$C', l['ms_per_step'], l['phases_ms']['numeric'], l['roofline']['frac'])"
  done
done
