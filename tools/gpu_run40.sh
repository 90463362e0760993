set -x
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -c "import paper_2106_12863_b200" || exit 1
B="timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu --no-e2e --no-comparator --no-parse --config c5"
for rep in 1 2; do
SINET_LIB_VARIANT=v3 $B > gpurun_out/r40_c5_v3_$rep.txt 2>&1
$B > gpurun_out/r40_c5_v7_$rep.txt 2>&1
SINET_LIB_VARIANT=v7b $B > gpurun_out/r40_c5_v7b_$rep.txt 2>&1
done
SINET_LIB_VARIANT=v7b timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 -k "inline or table_encodings" > gpurun_out/r40_pytest_v7b.txt 2>&1
for f in gpurun_out/r40_c*.txt; do python - "$f" <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[1], round(d['roofline']['kernel_ms'],4), round(d['ms_per_step'],4), round(d['roofline']['frac'],4), d['clocks']['sm_mhz'])
except Exception as e: print(sys.argv[1], 'ERR', e)
PY
done
tail -n 2 gpurun_out/r40_pytest_v7b.txt
