set -x
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -c "import paper_2106_12863_b200" || exit 1
B="timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --no-comparator --no-parse"
for v in main acc stcs accstcs; do
  if [ $v = main ]; then unset SINET_LIB_VARIANT; else export SINET_LIB_VARIANT=$v; fi
  $B > gpurun_out/r31_bench_c2_$v.txt 2>&1
  $B --config c4 --records-per-gpu 400000000 > gpurun_out/r31_bench_c4_$v.txt 2>&1
  $B --config c5 > gpurun_out/r31_bench_c5_$v.txt 2>&1
done
unset SINET_LIB_VARIANT
for r in 2 8; do SINET_RANGES=$r $B > gpurun_out/r31_bench_c2_ranges$r.txt 2>&1; SINET_RANGES=$r $B --config c4 --records-per-gpu 400000000 > gpurun_out/r31_bench_c4_ranges$r.txt 2>&1; done
tail -n 1 gpurun_out/r31_*.txt | cut -c1-300
