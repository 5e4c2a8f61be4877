#!/bin/bash
# A/B of HJMSV_PLANE schedules on one box: PLS="1 3" CFGS=3 bash tools/ab_schedules.sh
cd $GRAFT_REPO_ROOT
for pl in ${PLS:-1 3}; do
  echo "PLANE=$pl"; HJMSV_PLANE=$pl timeout 300 python tools/kprofile.py --configs ${CFGS:-3} --steps 20 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: print(l.strip()); continue
    print(d['config'], round(d['step_us'],1), d['kernels'])"
done
