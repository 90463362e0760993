#!/bin/bash
# One parameterised GPU job for gpurun:  gpurun -- bash tools/gpu_run.sh TAG STEP [STEP ...]
# Steps: smoke pytest pytest_merge pytest_new bench benchws ref c1..c5 shuf launches ncu_c2 ncu_c4 ncu_c5
#        ncu_ws ncu_ws_c4 san wscheck
# Every output lands in gpurun_out/TAG_<step>.txt (merged back by gpurun).
set -x
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
TAG=$1; shift
O=gpurun_out/${TAG}
python -c "import paper_2106_12863_b200" || exit 1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > ${O}_gpu.txt 2>&1
lscpu > ${O}_lscpu.txt 2>&1
# ncu reports are large (gpurun returns <= 64 MiB): keep CSV exports of the counters, the
# per-instruction source view and the details page, drop the .ncu-rep
export_rep() {
  ncu -i $1.ncu-rep --page raw --csv > $1_raw.csv 2>&1
  ncu -i $1.ncu-rep --page source --csv --print-source=sass > $1_src.csv 2>&1
  ncu -i $1.ncu-rep --page details > $1_details.txt 2>&1
  rm -f $1.ncu-rep
}
B="timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --no-comparator --no-parse"
for s in "$@"; do
  case $s in
    smoke) timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" > ${O}_smoke.txt 2>&1 ;;
    pytest) timeout 2400 python -m pytest tests -m gpu -q -x --timeout 1200 > ${O}_pytest_gpu.txt 2>&1 ;;
    pytest_merge) timeout 900 python -m pytest tests/test_gpu_merge.py -m gpu -q --timeout 300 > ${O}_pytest_merge.txt 2>&1 ;;
    bench) timeout 1200 python bench.py > ${O}_bench.txt 2>&1 ;;
    ref) timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > ${O}_ref.txt 2>&1 ;;
    c1|c2|c3|c4|c5) $B --config $s > ${O}_$s.txt 2>&1 ;;
    knob_*) # knob_NAME=VALUE_CFG: the bench line with one sinet_set_knob setting
      v=${s#knob_}; kv=${v%_*}; cfg=${v##*_}
      $B --config $cfg --knob $kv > ${O}_$s.txt 2>&1 ;;
    shufvar_*) # shufvar_NAME_CFG: the shuffled-order bench line with libsinet.NAME.so
      v=${s#shufvar_}; name=${v%_*}; cfg=${v##*_}
      SINET_LIB_VARIANT=$name $B --config $cfg --order shuffled --legs none > ${O}_$s.txt 2>&1 ;;
    shuf_cfg_*) cfg=${s#shuf_cfg_}; $B --config $cfg --order shuffled --legs none > ${O}_$s.txt 2>&1 ;;
    var_*) # var_NAME_CFG: the same bench line with libsinet.NAME.so (tools/build_variant.py)
      v=${s#var_}; name=${v%_*}; cfg=${v##*_}
      SINET_LIB_VARIANT=$name $B --config $cfg > ${O}_$s.txt 2>&1 ;;
    shuf) $B --order shuffled > ${O}_shuf.txt 2>&1 ;;
    shuf_c4) $B --config c4 --order shuffled > ${O}_shuf_c4.txt 2>&1 ;;
    launches) timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:^k_ -c 400 --csv --log-file ${O}_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-comparator --no-parse > ${O}_launches_run.txt 2>&1 ;;
    launches_shuf) timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:^k_ -c 200 --csv --log-file ${O}_launches_shuf.csv python bench.py --order shuffled --steps 2 --warmup 3 --legs none --no-cpu --no-e2e --no-comparator --no-parse > ${O}_launches_shuf_run.txt 2>&1 ;;
    ncu_part) timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_part -s 5 -c 5 -o ${O}_prof_part python bench.py --order shuffled --steps 1 --warmup 1 --profile > ${O}_ncu_part_run.txt 2>&1; for f in ${O}_prof_part*.ncu-rep; do export_rep ${f%.ncu-rep}; done ;;
    ncu_c2) timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_hist_stream -s 2 -c 1 -o ${O}_prof_c2 python bench.py --steps 2 --warmup 1 --profile > ${O}_ncu_c2_run.txt 2>&1; export_rep ${O}_prof_c2 ;;
    ncu_c4) timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_hist_stream -s 2 -c 1 -o ${O}_prof_c4 python bench.py --config c4 --steps 2 --warmup 1 --profile > ${O}_ncu_c4_run.txt 2>&1; export_rep ${O}_prof_c4 ;;
    ncu_c5) timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_hist_stream -s 2 -c 1 -o ${O}_prof_c5 python bench.py --config c5 --steps 2 --warmup 1 --profile > ${O}_ncu_c5_run.txt 2>&1; export_rep ${O}_prof_c5 ;;
    san) for t in memcheck racecheck synccheck; do timeout 900 compute-sanitizer --tool $t python tools/sanitize_case.py > ${O}_san_$t.txt 2>&1; done ;;
    wscheck) timeout 400 python tools/ws_check.py > ${O}_wscheck.txt 2>&1 ;;
    ab) timeout 900 python tools/ab_stream.py > ${O}_ab.txt 2>&1 ;;
    pytest_stream) timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -q -x --timeout 300 -k "not ws and (test_adversarial_parity or table_enc or inline or dense or bursty or gaps or c1_full or chunked or watchlist or (full_size_digest and stream))" > ${O}_pytest_stream.txt 2>&1 ;;
    pytest_part) timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -q -x --timeout 300 -k "partitioned or (full_size_digest and shuffled and (c1 or c2 or c5))" > ${O}_pytest_part.txt 2>&1 ;;
    pytest_range) timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q -x --timeout 300 -k "range_count" > ${O}_pytest_range.txt 2>&1 ;;
    pytest_new) timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -q --timeout 300 -k "ws or partitioned or bursty or gaps or dense or c1_full or table_enc or inline" > ${O}_pytest_new.txt 2>&1 ;;
    ncu_ws) timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_hist_ws -s 2 -c 1 -o ${O}_prof_ws python bench.py --steps 2 --warmup 1 --profile --knob stream_kernel=2 > ${O}_ncu_ws_run.txt 2>&1 ;;
    ncu_ws_c4) timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_hist_ws -s 2 -c 1 -o ${O}_prof_ws_c4 python bench.py --config c4 --steps 2 --warmup 1 --profile --knob stream_kernel=2 > ${O}_ncu_ws_c4_run.txt 2>&1 ;;
    atomshuf) timeout 600 python bench.py --order shuffled --legs none --knob shuffled_kernel=1 --no-cpu --no-e2e --no-comparator --no-parse > ${O}_atomshuf.txt 2>&1 ;;
    benchshuf) timeout 1200 python bench.py --order shuffled --legs c4@shuffled --no-cpu --no-e2e --no-comparator --no-parse > ${O}_benchshuf.txt 2>&1 ;;
    benchws) timeout 1800 python bench.py --knob stream_kernel=2 > ${O}_benchws.txt 2>&1 ;;
    *) echo "unknown step $s" ;;
  esac
done
tail -n 3 ${O}_*.txt | cut -c1-400
