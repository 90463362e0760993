set -x
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -c "import paper_2106_12863_b200" || exit 1
B="timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu --no-e2e --no-comparator --no-parse"
for rep in 1 2; do
for v in base kh6 kh8 kh9; do
  if [ $v = base ]; then $B > gpurun_out/r46_c2_${v}_$rep.txt 2>&1; else SINET_LIB_VARIANT=$v $B > gpurun_out/r46_c2_${v}_$rep.txt 2>&1; fi
done; done
for v in base kh6 kh8 kh9; do
  if [ $v = base ]; then $B --config c4 --records-per-gpu 400000000 > gpurun_out/r46_c4_${v}.txt 2>&1; else SINET_LIB_VARIANT=$v $B --config c4 --records-per-gpu 400000000 > gpurun_out/r46_c4_${v}.txt 2>&1; fi
done
for f in gpurun_out/r46_c*.txt; do python - "$f" <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[1], round(d['roofline']['kernel_ms'],4), round(d['ms_per_step'],4), round(d['roofline']['frac'],4), d['clocks']['sm_mhz'])
except Exception as e: print(sys.argv[1], 'ERR', e)
PY
done
