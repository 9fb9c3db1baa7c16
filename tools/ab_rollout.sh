# A/B of the fused rollout: bench.py with and without it, then the rollout
# kernel variants in variants/ (tools/build_variant.py) at S=10.
for sc in "simple_spread" "transport" "transport --envs 1000000"; do
  for m in "" "--per-step"; do
    python bench.py --scenario $sc --steps 40 --warmup 5 --no-cpu $m 2>&1 | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read());r=d['roofline']
print('$sc $m', 'value', d['value'], 'ms/step', d['ms_per_step'], 'kernel', r['kernel_ms'], 'frac', r['frac'], 'fused', d['fused_rollout'], 'e2e', d['e2e']['value'])"
  done
done
if ls variants/*.so >/dev/null 2>&1; then
  SWEEP_S=10 SWEEP_WORKLOADS=simple_spread,transport SWEEP_ENVS=transport=1000000 \
    python tools/sweep_variants.py paper_2207_03530_b200/libswarmsim_b200.so variants/*.so
  SWEEP_S=1 SWEEP_WORKLOADS=simple_spread,transport SWEEP_ENVS=transport=1000000 \
    python tools/sweep_variants.py paper_2207_03530_b200/libswarmsim_b200.so
fi
