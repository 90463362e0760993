set -x
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -c "import paper_2106_12863_b200" || exit 1
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 240 -k "not c2_full" > gpurun_out/pytest_gpu.txt 2>&1
for r in 1 2 3 6; do SINET_RANGES=$r timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --no-comparator > gpurun_out/bench_c2_r$r.txt 2>&1; done
for r in 1 3 6; do SINET_RANGES=$r timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --no-comparator --config c4 --records-per-gpu 400000000 > gpurun_out/bench_c4_r$r.txt 2>&1; done
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --no-comparator --config c5 --records-per-gpu 100000000 > gpurun_out/bench_c5.txt 2>&1
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --no-comparator --order shuffled > gpurun_out/bench_c2_shuf.txt 2>&1
tail -n 3 gpurun_out/*.txt
