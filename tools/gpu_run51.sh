set -x
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" > gpurun_out/r51_smoke.txt 2>&1
timeout 600 compute-sanitizer --tool initcheck python tools/sanitize_dense.py > gpurun_out/r51_dense_initcheck.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q -x --timeout 900 > gpurun_out/r51_pytest_gpu.txt 2>&1
timeout 600 python bench.py --no-cpu > gpurun_out/r51_bench_default.txt 2>&1
tail -n 3 gpurun_out/r51_*.txt | cut -c1-300
