# Session state check: HEAD check + CUPTI step timelines of the small/medium configs.
TAG=${1:-s7}
bash scripts/gpu_head_check.sh $TAG
for c in C1 C3 C4 C2-16384; do
  timeout 300 python scripts/step_timeline_probe.py $c > gpurun_out/timeline_${TAG}_$c.txt 2>&1; echo "timeline $c rc=$?"
done
