#!/bin/bash
# A/B of environment switches on one box, per-kernel timeline per config:
#   VARS="HJMSV_PFA=0 HJMSV_PFA=148" CFGS=3,1 bash tools/ab_env.sh
cd $GRAFT_REPO_ROOT
for vv in ${VARS:-X=0}; do
  echo "== $vv"
  env $vv timeout 600 python tools/kprofile.py --configs ${CFGS:-3} --steps ${STEPS:-40} 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: print(l.strip()); continue
    print(d['config'], 'step_us', round(d['step_us'],1), [(k[0][:14], k[1]) for k in d['kernels']])"
done
