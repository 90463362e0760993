set -x
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu.txt 2>&1
nproc >> gpurun_out/gpu.txt; lscpu | grep -E "Model name|^CPU\(s\)" >> gpurun_out/gpu.txt
timeout 120 ./tools/microbench > gpurun_out/microbench.txt 2>&1
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q -k "not c2_full" > gpurun_out/pytest_gpu.txt 2>&1
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.txt 2>&1
tail -5 gpurun_out/*.txt
