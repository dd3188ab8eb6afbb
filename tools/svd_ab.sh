#!/bin/bash
# A/B of library variants varlib/lib_<name>.so on the C2/C3 SVD times (tools/svd_times.py); run on a B200.
for v in "$@"; do
  cp varlib/lib_$v.so paper_1804_07531_b200/librsvd.so
  echo "== $v"
  timeout 300 python tools/svd_times.py C2 C3 2>/dev/null | python -c "
import sys, json
for l in sys.stdin:
    try: d = json.loads(l)
    except Exception: continue
    print(d['config'], d['alg'], d['v'], round(d['svd_ms'], 4))"
done
