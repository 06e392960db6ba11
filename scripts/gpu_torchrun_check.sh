# Path check of bench.py's N>1 branch through torchrun on ONE GPU: 2 ranks share the B200, the
# collectives are host-staged gloo (QM_DIST_BACKEND=gloo), peers mapped through CUDA IPC. Timings
# are meaningless (the ranks time-slice one GPU); this checks the multi-GPU step runs end to end.
mkdir -p gpurun_out
for C in C4 C2-131072 C5-64; do
  QM_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 --config $C --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/tr2_$C.log 2>&1; echo "torchrun $C rc=$?"
  grep '^{' gpurun_out/tr2_$C.log | tail -1 | python -c "
import json,sys; l=json.loads(sys.stdin.read()); print(l['config']['workload'], l['n_gpus'], l['value'], l['ms_per_step'], l['distributed'])"
done
