# A/B of an environment switch on bench lines: bash scripts/gpu_ab.sh VAR "v1 v2" "C3 C1" TAG
VAR=$1; VALS=$2; CFGS=$3; TAG=${4:-ab}
mkdir -p gpurun_out
for c in $CFGS; do for v in $VALS; do for rep in 1 2; do
  env $VAR=$v python bench.py --config $c --steps 20 --warmup 5 --no-e2e --no-cpu > gpurun_out/ab_${TAG}_${c}_${v}_$rep.log 2>&1
  python - "$c" "$v" "$rep" "gpurun_out/ab_${TAG}_${c}_${v}_$rep.log" <<'PY'
import json, sys
c, v, rep, f = sys.argv[1:]
line = [l for l in open(f) if l.startswith("{")][-1]
d = json.loads(line)
print(f"{c} {v} rep{rep}: step {d['ms_per_step']:.4f} ms numeric {d['phases_ms']['numeric']:.4f} ms frac {d['roofline']['frac']}")
PY
done; done; done
