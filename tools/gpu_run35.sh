set -x
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -c "import paper_2106_12863_b200" || exit 1
python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" > gpurun_out/r35_smoke.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q -x --timeout 900 > gpurun_out/r35_pytest_gpu.txt 2>&1
timeout 600 python bench.py > gpurun_out/r35_bench_default.txt 2>&1
tail -n 2 gpurun_out/r35_*.txt | cut -c1-400
