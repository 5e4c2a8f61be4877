#!/bin/bash
# One evidence round on a B200 (run under gpurun): the GPU suite, then bench lines for configs
# 0-4 + the reference arm, the ncu launch list of config 3, DRAM bytes per pass for every
# config and one --set full capture (tools/prof_r2.sh).   ROUND=r2h bash tools/evidence_round.sh
cd $GRAFT_REPO_ROOT
R=${ROUND:-r2h}
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${R}_pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/${R}_pytest_gpu.log
ROUND=$R bash tools/prof_r2.sh
