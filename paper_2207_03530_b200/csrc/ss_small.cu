// ss_small.cu — launch_small: fills the SmallArgs of a thread-per-env fused
// step from the world descriptor and dispatches to the kernel family's
// launcher (ss_spread.cu, ss_transport.cu, ss_catalog.cu, ss_flocking.cu).
#include "ss_small.cuh"

namespace ss {

int launch_small(World& w, const SsBuffers* buf, const SsStepIO* io, cudaStream_t st) {
  SmallArgs a;
  memset(&a, 0, sizeof(a));
  a.s = make_state(w, buf);
  a.ph = make_phys(w);
  a.ents = w.d_ents;
  a.pairs = w.d_pairs;
  const int NA = w.d.n_agents;
  if (NA < 1 || NA > kSmallMaxAgents) {
    set_error("fused kernel instantiated for 1.." + std::to_string(kSmallMaxAgents) + " agents");
    return SS_ERR_UNSUPPORTED;
  }
  if (io->mode & SS_DO_PHYSICS) {
    for (int i = 0; i < NA; ++i) a.act[i] = reinterpret_cast<const float2*>(io->actions[i]);
  }
  a.obs = io->obs;
  a.obs_stride = io->obs_agent_stride;
  a.rew = io->rew;
  a.done = io->done;
  a.mode = io->mode;
  a.raw_forces = io->raw_forces;
  a.obs_dim = w.d.obs_dim;
  a.guard = io->guard;
  a.guard_n = io->guard_count > 0 ? io->guard_count : 1;
  memcpy(a.sc, w.d.sc, sizeof(a.sc));
  memcpy(a.sd, w.d.sd, sizeof(a.sd));
  memcpy(a.si, w.d.si, sizeof(a.si));
  a.E = w.d.n_entities;
  a.P = w.d.n_pairs;
  switch (w.d.scenario) {
    case SS_SCN_SIMPLE_SPREAD: return launch_spread(w, a, st);
    case SS_SCN_TRANSPORT: return launch_transport(w, a, st);
    case SS_SCN_DROPOUT: return launch_dropout(w, a, st);
    case SS_SCN_WHEEL:
    case SS_SCN_GIVE_WAY:
    case SS_SCN_PASSAGE:
    case SS_SCN_BALANCE:
    case SS_SCN_WATERFALL:
    case SS_SCN_FOOTBALL: return launch_catalog(w, a, st);
    case SS_SCN_FLOCKING: return launch_flocking(w, a, st);
    default:
      set_error("launch_small: not a small scenario");
      return SS_ERR_SCENARIO;
  }
}

}  // namespace ss
