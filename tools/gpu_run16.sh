set -x
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -c "import paper_2106_12863_b200" || exit 1
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 300 -k "not full_size" > gpurun_out/pytest_gpu.txt 2>&1
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --no-comparator > gpurun_out/bench_c2.txt 2>&1
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --no-comparator --config c4 --records-per-gpu 400000000 > gpurun_out/bench_c4.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 900 -k "full_size" > gpurun_out/pytest_full.txt 2>&1
timeout 600 compute-sanitizer --tool racecheck python tools/sanitize_case.py > gpurun_out/san_racecheck.txt 2>&1
tail -n 3 gpurun_out/*.txt
