set -x
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -c "import paper_2106_12863_b200" || exit 1
B="timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --no-comparator --no-parse"
$B > gpurun_out/r32_bench_c2.txt 2>&1
$B --config c4 --records-per-gpu 400000000 > gpurun_out/r32_bench_c4.txt 2>&1
$B --config c5 > gpurun_out/r32_bench_c5.txt 2>&1
$B --config c3 > gpurun_out/r32_bench_c3_1gpu.txt 2>&1
$B --config c1 > gpurun_out/r32_bench_c1.txt 2>&1
$B --order shuffled > gpurun_out/r32_bench_c2_shuffled.txt 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 -k "not full_size" > gpurun_out/r32_pytest_gpu.txt 2>&1
tail -n 1 gpurun_out/r32_*.txt | cut -c1-300
