# A/B of experimental library builds (scripts/build_variants.py) on bench lines.
# Usage: bash scripts/gpu_lib_ab.sh "base v1 v2" "C3 C2-131072" TAG [REPS]
NAMES=$1; CFGS=$2; TAG=${3:-lab}; REPS=${4:-2}
mkdir -p gpurun_out
for c in $CFGS; do for rep in $(seq $REPS); do for v in $NAMES; do
  QM_LIB_PATH=exp_lib/libqmb200_$v.so timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/lab_${TAG}_${c}_${v}_$rep.log 2>&1 || echo "bench $c $v failed"
  python - "$c" "$v" "$rep" "gpurun_out/lab_${TAG}_${c}_${v}_$rep.log" <<'PY'
import json, sys
c, v, rep, f = sys.argv[1:]
try:
    line = [l for l in open(f) if l.startswith("{")][-1]
    d = json.loads(line)
    print(f"{c} {v} rep{rep}: step {d['ms_per_step']:.4f} ms numeric {d['phases_ms']['numeric']:.4f} ms frac {d['roofline']['frac']} clk {d['clocks']['sm_mhz']}")
except Exception as e:
    print(c, v, rep, "parse failed", e)
PY
done; done; done
