#!/bin/bash
# usage: tools/gpu_check.sh [tests] [bench] [ncu_list] [ncu_full <kernel-regex>]
set -u
mkdir -p gpurun_out
for what in "$@"; do
  case $what in
    tests) timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu --maxfail=20 -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "tests_rc=$?"; grep -E "passed|failed|FAILED" gpurun_out/gpu_tests.log | tail -25 ;;
    smoke) timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke_rc=$?"; tail -4 gpurun_out/smoke.log ;;
    bench) timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.log 2>&1; echo "bench_rc=$?"; tail -c 3000 gpurun_out/bench.log ;;
    ncu_list) timeout 300 python tools/one_step.py C2 2 > gpurun_out/one_step.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv python tools/one_step.py C2 2 > gpurun_out/ncu.log 2>&1; echo "ncu_list_rc=$?" ;;
  esac
done
