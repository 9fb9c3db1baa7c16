#!/usr/bin/env bash
# One ncu --set full capture of a fused step kernel in steady state (GPU box, 1 GPU):
#   bash tools/prof_one.sh SCENARIO KERNEL_REGEX [PRESTEPS]
# runs the step loop plainly first, then under ncu skipping PRESTEPS launches.
set -u
OUT=gpurun_out; mkdir -p $OUT
S=$1; K=$2; PRE=${3:-1}
CMD="python tools/step_loop.py $S 0 $((PRE + 2))"
$CMD > $OUT/plain_$S.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:$K -s $PRE -c 1 \
  -o $OUT/full_$S $CMD > $OUT/ncu_full_$S.log 2>&1
echo "ncu: $?"
python tools/ncu_summary.py $OUT/full_$S.ncu-rep $OUT/full_$S && rm -f $OUT/full_$S.ncu-rep
