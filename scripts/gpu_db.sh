# Double-buffered epilogue (Tma64d): parity, then A/B against the plain Tma64 (QM_EPILOGUE_DB=0).
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/t_db.log 2>&1; echo "parity rc=$?"; tail -2 gpurun_out/t_db.log
for c in C3 C2-16384 C1; do for rep in 1 2; do for db in 1 0; do
  QM_EPILOGUE_DB=$db timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu 2>/dev/null | tail -1 | python -c "
import json,sys; l=json.loads(sys.stdin.read()); print('$c db=$db', l['phases_ms'], round(l['roofline']['achieved'],2), round(l['roofline']['frac'],4))"
done; done; done
