#!/usr/bin/env bash
# One gpurun call: GPU tests, a bench line per BASELINE config (plus 1M-env
# transport / flocking), the reference arm per config, the ncu launch list of
# the default bench command.  Results land in gpurun_out/ (copy what is to be
# judged into profiles/r02/).
set -u
OUT=gpurun_out
mkdir -p $OUT
python -m pytest tests -m gpu -q 2>&1 | grep -v "^  " | tail -30 > $OUT/re_tests.log
for s in simple_spread transport flocking dispersion discovery; do
  python bench.py --scenario $s --steps 20 --warmup 5 > $OUT/re_bench_$s.json 2> $OUT/re_bench_$s.err
  python bench.py --impl reference --scenario $s --steps 20 --warmup 5 > $OUT/re_ref_$s.json 2> $OUT/re_ref_$s.err
done
for s in transport flocking; do
  python bench.py --scenario $s --envs 1000000 --steps 20 --warmup 5 > $OUT/re_bench_${s}_1000000.json 2> /dev/null
done
python bench.py --scenario dispersion --strong --steps 10 --warmup 3 --no-cpu > $OUT/re_bench_dispersion_strong.json 2>/dev/null
BENCH="python bench.py --steps 10 --warmup 3 --soak 0 --no-cpu"
$BENCH > $OUT/re_plain.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
      --log-file $OUT/re_launches_simple_spread.csv $BENCH > $OUT/re_ncu_launches.log 2>&1
cat $OUT/re_tests.log
