set -u
OUT=gpurun_out
for s in transport flocking; do
  python bench.py --scenario $s --envs 1000000 --steps 20 --warmup 5 > $OUT/re_bench_${s}_1000000.json 2> /dev/null
done
ROLLOUT=10 bash tools/profile_all.sh simple_spread
ROLLOUT=10 bash tools/profile_all.sh transport
ROLLOUT=10 ENVS=1000000 bash tools/profile_all.sh transport
ENVS=1000000 bash tools/profile_all.sh transport
ls $OUT
