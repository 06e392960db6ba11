# C3 (about one triple per C block): numeric-phase variants and one ncu capture of k_numeric_tma.
TAG=${1:-c3}
mkdir -p gpurun_out
run() { timeout 300 env "$@" python bench.py --config C3 --steps 10 --warmup 3 --no-e2e --no-cpu 2>/dev/null | tail -1 | python -c "
import json,sys; l=json.loads(sys.stdin.read()); print('$*', l['phases_ms'], round(l['roofline']['achieved'],2), round(l['roofline']['frac'],4))"; }
run X=0
run QM_TMA_VARIANT=wide
run QM_UNIT_ORDER=k
run QM_CLAIM_AHEAD=0
run QM_UNIT_ORDER=k QM_TMA_VARIANT=wide
bash scripts/gpu_ncu_numeric.sh $TAG C3
ncu -i gpurun_out/prof_${TAG}_C3.ncu-rep --page raw --csv > gpurun_out/ncu_raw_${TAG}_C3.csv 2>/dev/null
ncu -i gpurun_out/prof_${TAG}_C3.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu_src_${TAG}_C3.csv 2>/dev/null
ls -la gpurun_out/prof_${TAG}_C3.ncu-rep
