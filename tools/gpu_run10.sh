set -x
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -c "import paper_2106_12863_b200" || exit 1
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 240 -k "not c2_full" > gpurun_out/pytest_gpu.txt 2>&1
SINET_STREAM_THREADS=1024 timeout 1200 python -m pytest tests -m gpu -q -x --timeout 240 -k "not c2_full" > gpurun_out/pytest_gpu_1024.txt 2>&1
for th in 512 1024; do for g in 1 2; do SINET_STREAM_THREADS=$th SINET_STREAM_GROUPS=$g timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --no-comparator > gpurun_out/bench_c2_t${th}_g$g.txt 2>&1; done; done
for th in 512 1024; do SINET_STREAM_THREADS=$th timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --no-comparator --config c4 --records-per-gpu 400000000 > gpurun_out/bench_c4_t$th.txt 2>&1; done
SINET_STREAM_THREADS=1024 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_hist_stream -s 2 -c 1 -o gpurun_out/prof_stream10 python bench.py --steps 2 --warmup 1 --profile > gpurun_out/ncu_full_run.txt 2>&1
tail -n 3 gpurun_out/*.txt
