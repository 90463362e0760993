set -x
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -c "import paper_2106_12863_b200" || exit 1
for v in main sel intrin selintrin; do
  if [ $v = main ]; then unset SINET_LIB_VARIANT; else export SINET_LIB_VARIANT=$v; fi
  timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --no-comparator --no-parse > gpurun_out/r30_bench_c2_$v.txt 2>&1
  timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --no-comparator --no-parse --config c4 --records-per-gpu 400000000 > gpurun_out/r30_bench_c4_$v.txt 2>&1
done
unset SINET_LIB_VARIANT
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 -k "not full_size" > gpurun_out/r30_pytest_gpu.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_hist_stream -s 2 -c 1 -o gpurun_out/r30_prof_stream python bench.py --steps 2 --warmup 1 --profile > gpurun_out/r30_ncu_full_run.txt 2>&1
tail -n 3 gpurun_out/r30_*.txt
