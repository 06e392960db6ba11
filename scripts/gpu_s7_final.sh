# Final check of the session: GPU suite, smoke, C5-32 / C3 / C1 lines (kernel names), default line + reference arm.
TAG=${1:-h4}
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu_$TAG.log
timeout 300 python __graft_entry__.py --smoke > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke_$TAG.log
for C in C5-32 C3 C1; do timeout 900 python bench.py --config $C --steps 10 --warmup 3 --no-e2e --no-cpu 2>/dev/null | tail -1 > gpurun_out/bench_${TAG}_$C.json; python -c "
import json; d=json.load(open('gpurun_out/bench_${TAG}_$C.json')); print('$C', d['ms_per_step'], d['phases_ms'], d['roofline']['kernel'], d['roofline']['frac'], d['roofline']['traffic'])"; done
timeout 900 python bench.py > gpurun_out/bench_$TAG.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench_$TAG.log | cut -c1-400
timeout 600 python bench.py --impl reference > gpurun_out/benchref_$TAG.log 2>&1; echo "benchref rc=$?"; tail -1 gpurun_out/benchref_$TAG.log | cut -c1-200
