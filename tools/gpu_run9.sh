set -x
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 600 compute-sanitizer --tool memcheck --show-backtrace device python tools/watch_case.py > gpurun_out/san_watch.txt 2>&1
tail -n 40 gpurun_out/san_watch.txt
