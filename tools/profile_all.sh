#!/usr/bin/env bash
# Profiling runs for profiles/ (execute on the GPU box via gpurun, 1 GPU; one
# ncu invocation per gpurun call):
#   bash tools/profile_all.sh launches     bench plainly, then its ncu launch list
#   [ENVS=n] [ROLLOUT=S] bash tools/profile_all.sh SCENARIO   step loop plainly, then one
#                                          ncu --set full capture of the fused kernel in steady
#                                          state (ENVS: batch size, default the workload's;
#                                          ROLLOUT: capture the S-step rollout kernel instead)
# Summaries land in gpurun_out/ (tools/ncu_summary.py); the .ncu-rep is deleted
# to keep the merge-back small.
set -u
OUT=gpurun_out
mkdir -p $OUT
what=${1:-launches}
if [ "$what" = launches ]; then
  BENCH="python bench.py --steps 10 --warmup 3 --soak 0 --no-cpu"
  $BENCH > $OUT/plain_bench.log 2>&1 && \
    ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
        --log-file $OUT/launches_simple_spread.csv $BENCH > $OUT/ncu_launches.log 2>&1
  echo "launches: $?"
  exit 0
fi
declare -A KERN=([simple_spread]=k_simple_spread [transport]=k_transport [flocking]=k_flocking_w \
                 [dispersion]=k_dispersion [discovery]=k_discovery)
# launches skipped before the capture: steady state (flocking's agents
# gather at the beacon after ~1k steps; the others settle within tens)
declare -A PRE=([simple_spread]=20 [transport]=200 [flocking]=1500 [dispersion]=20 [discovery]=50)
s=$what
ENVS=${ENVS:-0}
tag=$s${ENVS/#0/}
[ "$ENVS" != 0 ] && tag=${s}_$ENVS
ROLLOUT=${ROLLOUT:-0}
kern=${KERN[$s]}
pre=${PRE[$s]}
if [ "$ROLLOUT" != 0 ]; then
  kern=${kern}_rollout
  pre=$(( (pre + ROLLOUT - 1) / ROLLOUT ))
  tag=${s}_rollout${ROLLOUT}${ENVS/#0/}
  [ "$ENVS" != 0 ] && tag=${s}_rollout${ROLLOUT}_$ENVS
fi
CMD="python tools/step_loop.py $s $ENVS $((pre + 2)) $ROLLOUT"
$CMD > $OUT/plain_$tag.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:$kern -s $pre -c 1 \
      -o $OUT/full_$tag $CMD > $OUT/ncu_full_$tag.log 2>&1
echo "$tag: $?"
[ -f $OUT/full_$tag.ncu-rep ] && python tools/ncu_summary.py $OUT/full_$tag.ncu-rep $OUT/full_$tag && rm -f $OUT/full_$tag.ncu-rep
exit 0
