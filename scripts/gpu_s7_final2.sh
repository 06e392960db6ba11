# Final check + refreshed sweep lines (the symbolic phase changed for the small-key-space configs).
TAG=${1:-h5}
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu_$TAG.log
timeout 300 python __graft_entry__.py --smoke > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke_$TAG.log
for C in C1 C2-16384 C2-32768 C2-65536 C2-131072 C3 C4 C5-32 C5-128; do timeout 900 python bench.py --config $C --steps 10 --warmup 3 --no-e2e --no-cpu 2>/dev/null | tail -1 > gpurun_out/bench_${TAG}_$C.json; python -c "
import json; d=json.load(open('gpurun_out/bench_${TAG}_$C.json')); print('$C', d['ms_per_step'], d['phases_ms'], round(d['value']), d['roofline']['kernel'], d['roofline']['achieved'], d['roofline']['frac'], d['clocks']['sm_mhz'], d['clocks']['reasons'])"; done
timeout 900 python bench.py > gpurun_out/bench_$TAG.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench_$TAG.log | cut -c1-300
timeout 600 python bench.py --impl reference > gpurun_out/benchref_$TAG.log 2>&1; echo "benchref rc=$?"; tail -1 gpurun_out/benchref_$TAG.log | cut -c1-200
