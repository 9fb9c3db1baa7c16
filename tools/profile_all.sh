#!/usr/bin/env bash
# Profiling run for profiles/ (execute on the GPU box via gpurun, 1 GPU):
#   1. the bench command plainly, then its ncu launch list (per-launch times)
#   2. per workload: the step loop plainly, then one ncu --set full capture of
#      the fused step kernel (ncu only after the same command exited 0).
set -u
OUT=gpurun_out
mkdir -p $OUT
BENCH="python bench.py --steps 10 --warmup 3 --soak 0 --no-cpu"
$BENCH > $OUT/plain_bench.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
      --log-file $OUT/launches_simple_spread.csv $BENCH > $OUT/ncu_launches.log 2>&1
declare -A KERN=([simple_spread]=k_simple_spread [transport]=k_transport [flocking]=k_flocking \
                 [dispersion]=k_dispersion [discovery]=k_discovery)
for s in simple_spread transport flocking dispersion discovery; do
  CMD="python tools/step_loop.py $s 0 3"
  $CMD > $OUT/plain_$s.log 2>&1 && \
    ncu --set full --clock-control none --import-source on -k regex:${KERN[$s]} -s 1 -c 1 \
        -o $OUT/full_$s $CMD > $OUT/ncu_full_$s.log 2>&1
  echo "$s: $?"
done
# keep gpurun_out small: summaries only
for s in simple_spread transport flocking dispersion discovery; do
  [ -f $OUT/full_$s.ncu-rep ] && python tools/ncu_summary.py $OUT/full_$s.ncu-rep $OUT/full_$s && rm -f $OUT/full_$s.ncu-rep
done
