set -x
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -c "import paper_2106_12863_b200" || exit 1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 300 > gpurun_out/pytest_gpu.txt 2>&1
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_full.txt 2>&1
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_hist|k_materialize|k_add" --csv --log-file gpurun_out/launches11.csv python bench.py --steps 5 --warmup 1 --profile > gpurun_out/ncu_launch_run.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_hist_stream -s 2 -c 1 -o gpurun_out/prof_stream11 python bench.py --steps 2 --warmup 1 --profile > gpurun_out/ncu_full_run.txt 2>&1
timeout 600 compute-sanitizer --tool memcheck python tools/sanitize_case.py > gpurun_out/san_memcheck.txt 2>&1
timeout 600 compute-sanitizer --tool racecheck python tools/sanitize_case.py > gpurun_out/san_racecheck.txt 2>&1
timeout 600 compute-sanitizer --tool synccheck python tools/sanitize_case.py > gpurun_out/san_synccheck.txt 2>&1
tail -n 3 gpurun_out/*.txt
