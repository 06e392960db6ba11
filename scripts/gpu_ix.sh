# Cached row index: parity (all GPU tests of the symbolic / parity files), then A/B of step times.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_partition.py -x -q > gpurun_out/t_ix.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/t_ix.log
for c in C1 C3 C2-16384 C4 C2-131072; do for ix in 1 0; do
  QM_ROW_INDEX=$ix timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu 2>/dev/null | tail -1 | python -c "
import json,sys; l=json.loads(sys.stdin.read()); print('$c ix=$ix step', l['ms_per_step'], l['phases_ms'], l['value'], l.get('operand_metadata',{}).get('row_index'))"
done; done
