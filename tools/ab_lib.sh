#!/bin/bash
# A/B of library builds on one box, per-kernel device timeline per config:
#   LIBS="lib/variants/a.so lib/variants/b.so" CFGS=3,1,2,4 bash tools/ab_lib.sh
cd $GRAFT_REPO_ROOT
for rep in 1 2; do
for L in ${LIBS}; do
  echo "== $L (pass $rep)"
  HJMSV_LIB=$L timeout 600 python tools/kprofile.py --configs ${CFGS:-3,1} --steps ${STEPS:-40} 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: print(l.strip()); continue
    print(d['config'], 'step_us', round(d['step_us'],1), [(k[0][:14], k[1]) for k in d['kernels']])"
done
done
