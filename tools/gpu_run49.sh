set -x
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 300 python tools/sanitize_dense.py > gpurun_out/r49_dense_plain.txt 2>&1
timeout 900 compute-sanitizer --tool racecheck python tools/sanitize_dense.py > gpurun_out/r49_dense_racecheck.txt 2>&1
timeout 600 compute-sanitizer --tool memcheck python tools/sanitize_dense.py > gpurun_out/r49_dense_memcheck.txt 2>&1
timeout 600 compute-sanitizer --tool synccheck python tools/sanitize_dense.py > gpurun_out/r49_dense_synccheck.txt 2>&1
tail -n 3 gpurun_out/r49_*.txt
