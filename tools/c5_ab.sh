#!/bin/bash
# A/B of library variants varlib/lib_<name>.so on the C5 subspace/Krylov SVD times; run on a B200.
for v in "$@"; do
  cp varlib/lib_$v.so paper_1804_07531_b200/librsvd.so
  echo "== $v"
  timeout 600 python tools/svd_times.py C5 2>/dev/null | python -c "
import sys, json
for l in sys.stdin:
    try: d = json.loads(l)
    except Exception: continue
    print(d['config'], d['alg'], d['v'], round(d['svd_ms'], 3))"
done
