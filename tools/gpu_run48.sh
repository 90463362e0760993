set -x
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -c "import paper_2106_12863_b200" || exit 1
python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" > gpurun_out/r48_smoke.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q -x --timeout 900 > gpurun_out/r48_pytest_gpu.txt 2>&1
timeout 600 python bench.py > gpurun_out/r48_bench_default.txt 2>&1
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r48_bench_ref.txt 2>&1
B="timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --no-comparator --no-parse"
$B --config c4 --records-per-gpu 400000000 > gpurun_out/r48_bench_c4.txt 2>&1
$B --config c5 > gpurun_out/r48_bench_c5.txt 2>&1
$B --config c1 > gpurun_out/r48_bench_c1.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r48_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-comparator --no-parse > gpurun_out/r48_ncu_launch_run.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_hist_stream -s 2 -c 1 -o gpurun_out/r48_prof_stream python bench.py --steps 2 --warmup 1 --profile > gpurun_out/r48_ncu_full_run.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_hist_stream -s 2 -c 1 -o gpurun_out/r48_prof_stream_c5 python bench.py --config c5 --steps 2 --warmup 1 --profile > gpurun_out/r48_ncu_full_c5_run.txt 2>&1
timeout 600 compute-sanitizer --tool memcheck python tools/sanitize_case.py > gpurun_out/r48_san_memcheck.txt 2>&1
timeout 900 compute-sanitizer --tool racecheck python tools/sanitize_case.py > gpurun_out/r48_san_racecheck.txt 2>&1
timeout 600 compute-sanitizer --tool synccheck python tools/sanitize_case.py > gpurun_out/r48_san_synccheck.txt 2>&1
tail -n 2 gpurun_out/r48_*.txt | cut -c1-300
