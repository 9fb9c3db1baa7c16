for envs in "transport=1000000" "transport=100000"; do
  for S in 1 10; do
    echo "envs=$envs S=$S"
    SWEEP_S=$S SWEEP_WORKLOADS=simple_spread,transport SWEEP_ENVS=$envs python tools/sweep_variants.py paper_2207_03530_b200/libswarmsim_b200.so variants/*.so
  done
done
