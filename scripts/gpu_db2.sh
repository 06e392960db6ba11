# Double-buffered epilogue A/B (occupancy check included).
for c in C3 C2-16384; do for db in 1 0; do
  QM_EPILOGUE_DB=$db timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu 2>/dev/null | tail -1 | python -c "
import json,sys; l=json.loads(sys.stdin.read()); print('$c db=$db', l['phases_ms'], round(l['roofline']['achieved'],2), round(l['roofline']['frac'],4))"
done; done
QM_EPILOGUE_DB=1 timeout 600 ncu --metrics launch__occupancy_limit_registers,launch__registers_per_thread,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active,gpu__time_duration.sum --clock-control none -k regex:k_numeric_tma -s 1 -c 1 python bench.py --config C3 --steps 1 --warmup 1 --no-e2e --no-cpu 2>&1 | grep -E "occupancy|registers|dmma|duration"
