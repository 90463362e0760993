set -x
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -c "import paper_2106_12863_b200" || exit 1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r20_smi.txt
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 600 > gpurun_out/r20_pytest_gpu.txt 2>&1
timeout 600 python bench.py > gpurun_out/r20_bench_default.txt 2>&1
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r20_bench_ref.txt 2>&1
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --no-comparator --config c4 --records-per-gpu 400000000 > gpurun_out/r20_bench_c4.txt 2>&1
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --no-comparator --config c5 > gpurun_out/r20_bench_c5.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r20_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-comparator > gpurun_out/r20_ncu_launch_run.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_hist_stream -s 2 -c 1 -o gpurun_out/r20_prof_stream python bench.py --steps 2 --warmup 1 --profile > gpurun_out/r20_ncu_full_run.txt 2>&1
tail -n 3 gpurun_out/r20_*.txt
