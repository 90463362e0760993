set -x
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
SINET_LIB_VARIANT=r4 timeout 300 python tools/sanitize_dense.py > gpurun_out/r50_r4_plain.txt 2>&1
SINET_LIB_VARIANT=r4 timeout 900 compute-sanitizer --tool racecheck python tools/sanitize_dense.py > gpurun_out/r50_r4_racecheck.txt 2>&1
SINET_LIB_VARIANT=r4 timeout 600 compute-sanitizer --tool initcheck python tools/sanitize_dense.py > gpurun_out/r50_r4_initcheck.txt 2>&1
tail -n 6 gpurun_out/r50_*.txt
