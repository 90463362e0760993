set -x
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -c "import paper_2106_12863_b200" || exit 1
B="timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu --no-e2e --no-comparator --no-parse"
for rep in 1 2; do
for v in base e1 e2 e12; do
  if [ $v = base ]; then $B > gpurun_out/r36_c2_${v}_$rep.txt 2>&1; else SINET_LIB_VARIANT=$v $B > gpurun_out/r36_c2_${v}_$rep.txt 2>&1; fi
done; done
$B --config c4 --records-per-gpu 400000000 > gpurun_out/r36_c4_base.txt 2>&1
SINET_LIB_VARIANT=e12 $B --config c4 --records-per-gpu 400000000 > gpurun_out/r36_c4_e12.txt 2>&1
$B --config c5 > gpurun_out/r36_c5_base.txt 2>&1
SINET_LIB_VARIANT=e12 $B --config c5 > gpurun_out/r36_c5_e12.txt 2>&1
SINET_LIB_VARIANT=e12 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 > gpurun_out/r36_pytest_e12.txt 2>&1
for f in gpurun_out/r36_c*.txt; do python - "$f" <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[1], round(d['roofline']['kernel_ms'],4), round(d['ms_per_step'],4), round(d['roofline']['frac'],4), d['clocks']['sm_mhz'])
except Exception as e: print(sys.argv[1], 'ERR', e)
PY
done
tail -n 2 gpurun_out/r36_pytest_e12.txt
