set -x
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -c "import paper_2106_12863_b200" || exit 1
B="timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu --no-e2e --no-comparator --no-parse"
for rep in 1 2; do
$B > gpurun_out/r47_c2_base_$rep.txt 2>&1
SINET_LIB_VARIANT=mm $B > gpurun_out/r47_c2_mm_$rep.txt 2>&1
done
$B --config c4 --records-per-gpu 400000000 > gpurun_out/r47_c4_base.txt 2>&1
SINET_LIB_VARIANT=mm $B --config c4 --records-per-gpu 400000000 > gpurun_out/r47_c4_mm.txt 2>&1
SINET_LIB_VARIANT=mm timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 -k "adversarial or dense_stream or bursty or gaps or c2_full or chunked or inline or watchlist or labelled" > gpurun_out/r47_pytest_mm.txt 2>&1
for f in gpurun_out/r47_c*.txt; do python - "$f" <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[1], round(d['roofline']['kernel_ms'],4), round(d['ms_per_step'],4), round(d['roofline']['frac'],4), d['clocks']['sm_mhz'])
except Exception as e: print(sys.argv[1], 'ERR', e)
PY
done
tail -n 2 gpurun_out/r47_pytest_mm.txt
