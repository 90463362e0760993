set -x
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -c "import paper_2106_12863_b200" || exit 1
timeout 900 python -m pytest tests/test_gpu_parse.py -q -x --timeout 600 > gpurun_out/r33_pytest_parse.txt 2>&1
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --no-comparator > gpurun_out/r33_bench_c2.txt 2>&1
SINET_LIB_VARIANT=p8 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --no-comparator > gpurun_out/r33_bench_c2_p8.txt 2>&1
SINET_LIB_VARIANT=p8 timeout 900 python -m pytest tests/test_gpu_parse.py -q -x --timeout 600 > gpurun_out/r33_pytest_parse_p8.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:parse -c 1 -o gpurun_out/r33_prof_parse python -m pytest tests/test_gpu_parse.py -q -k full_size > gpurun_out/r33_ncu_parse_run.txt 2>&1
tail -n 1 gpurun_out/r33_*.txt | cut -c1-300
