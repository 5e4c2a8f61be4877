#!/bin/bash
# A/B of diagnostic switches on one box: kernel times for config ${CFGS:-1}
cd $GRAFT_REPO_ROOT
for d in ${DBGS:-0 1 2 0}; do
  echo "DBG=$d"; HJMSV_DBG=$d timeout 300 python tools/kprofile.py --configs ${CFGS:-1} --steps 40 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: print(l.strip()); continue
    print(d['config'], round(d['step_us'],1), d['kernels'])"
done
