# Transport captures after the constant-descriptor change (per-step 1M and
# the 10-step rollout at 100k / 1M), then the 1M bench lines.
set -u
OUT=gpurun_out
ROLLOUT=10 bash tools/profile_all.sh transport
ROLLOUT=10 ENVS=1000000 bash tools/profile_all.sh transport
ENVS=1000000 bash tools/profile_all.sh transport
ROLLOUT=10 bash tools/profile_all.sh simple_spread
