// ss_capi.cu — the extern "C" boundary (include/swarmsim_b200.h).
#include <cstdio>
#include <cstdlib>
#include <new>

#include "ss_geometry.cuh"

namespace ss {

static thread_local std::string g_last_error;

void set_error(const std::string& msg) { g_last_error = msg; }

bool pdl_enabled() {
  static const bool on = std::getenv("SS_NO_PDL") == nullptr;
  return on;
}

int cuda_status(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return SS_OK;
  set_error(std::string(what) + ": " + cudaGetErrorString(e));
  return SS_ERR_CUDA;
}

int launch_small(World& w, const SsBuffers* buf, const SsStepIO* io, cudaStream_t st);
int launch_large(World& w, const SsBuffers* buf, const SsStepIO* io, cudaStream_t st);
int launch_rollout(World& w, const SsBuffers* buf, const SsRolloutIO* io, cudaStream_t st);
int launch_generic(World& w, const SsBuffers* buf, const SsStepIO* io, const uint64_t* decode_mask,
                   int* d_status, cudaStream_t st);
int launch_reset(World& w, const SsBuffers* buf, const uint8_t* mask, const int64_t* mask_base,
                 const int64_t* mask_total, cudaStream_t st);
int launch_mask_count(World& w, const uint8_t* mask, int64_t* count_out, cudaStream_t st);
int launch_check_actions(int n_agents, int64_t B, const float* const* actions, int* flag,
                         cudaStream_t st);
int launch_publish_flag(const int* flag, int* host_out, int n, cudaStream_t st);
int launch_check_sets(const float* const* bases, int n_sets, int A, int64_t agent_stride, int64_t n,
                      int* flags, cudaStream_t st);
int launch_collision_force(const float* pix, const float* piy, const float* pjx, const float* pjy,
                           float dmin, float sign, float ck, float k, float* fx, float* fy,
                           uint8_t* active, int64_t n, cudaStream_t st);
int launch_closest_points(const float* pos_i, const float* rot_i, ShapeK si, const float* pos_j,
                          const float* rot_j, ShapeK sj, float* out_i, float* out_j, int64_t n,
                          int* status, cudaStream_t st);
int launch_lidar(World& w, const SsBuffers* buf, int agent, const SsLidarDesc* lidar, float* out,
                 cudaStream_t st);
int launch_cast_ray(World& w, const SsBuffers* buf, int exclude, const float* ox, const float* oy,
                    const double* angle, double max_range, float* out, cudaStream_t st);
int launch_np_trig(const float* x, float* out, int64_t n, int want_cos, cudaStream_t st);

template <class T>
static int upload(const std::vector<T>& v, T** dst) {
  *dst = nullptr;
  if (v.empty()) return SS_OK;
  cudaError_t e = cudaMalloc(reinterpret_cast<void**>(dst), v.size() * sizeof(T));
  if (e != cudaSuccess) return cuda_status(e, "cudaMalloc (world tables)");
  e = cudaMemcpy(*dst, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice);
  return cuda_status(e, "cudaMemcpy (world tables)");
}

static void free_world(World* w) {
  if (!w) return;
  cudaFree(w->d_ents);
  cudaFree(w->d_pairs);
  cudaFree(w->d_reset_ops);
  cudaFree(w->d_lidar_dirs);
  cudaFree(w->d_scan);
  cudaFree(w->d_joints);
  delete w;
}

static int validate_desc(const SsWorldDesc* d) {
  if (!d) { set_error("null world descriptor"); return SS_ERR_CONTRACT; }
  if (d->abi_version != SS_ABI_VERSION) {
    set_error("ABI version mismatch: library " + std::to_string(SS_ABI_VERSION) + ", caller " +
              std::to_string(d->abi_version));
    return SS_ERR_CONTRACT;
  }
  if (d->batch < 1) { set_error("batch_size must be >= 1"); return SS_ERR_CONTRACT; }
  if (d->n_entities < 0 || d->n_entities > SS_MAX_ENTITIES) { set_error("bad entity count"); return SS_ERR_CONTRACT; }
  if (d->n_agents < 0 || d->n_agents > d->n_entities || d->n_agents > SS_MAX_AGENTS) {
    set_error("bad agent count"); return SS_ERR_CONTRACT;
  }
  if (d->global_batch < d->batch || d->env_offset < 0 || d->env_offset + d->batch > d->global_batch) {
    set_error("shard [env_offset, env_offset+batch) outside global_batch"); return SS_ERR_CONTRACT;
  }
  if (d->scenario < SS_SCN_PHYSICS_ONLY || d->scenario > SS_SCN_FOOTBALL) {
    set_error("unknown scenario id " + std::to_string(d->scenario)); return SS_ERR_SCENARIO;
  }
  if (d->n_reset_ops < 0 || d->n_reset_ops > SS_MAX_RESET_OPS) { set_error("bad reset program"); return SS_ERR_CONTRACT; }
  for (int k = 0; k < d->n_entities; ++k) {
    const SsEntityDesc& e = d->entities[k];
    if (e.shape < SS_SPHERE || e.shape > SS_LINE) {
      set_error("entity " + std::to_string(k) + " has an unsupported shape");
      return SS_ERR_SHAPE_PAIR;
    }
    const int rows = e.movable ? d->n_dyn : d->n_stat;
    if (e.slot < 0 || e.slot >= rows) { set_error("entity slot out of range"); return SS_ERR_CONTRACT; }
  }
  for (int p = 0; p < d->n_pairs; ++p) {
    const SsPairDesc& q = d->pairs[p];
    if (q.i < 0 || q.j <= q.i || q.j >= d->n_entities) { set_error("bad pair list"); return SS_ERR_CONTRACT; }
  }
  if (d->substeps < 1 || d->substeps > SS_MAX_SUBSTEPS) {
    set_error("substeps must be in [1, " + std::to_string(SS_MAX_SUBSTEPS) + "]"); return SS_ERR_CONTRACT;
  }
  if (d->n_joints < 0 || d->n_joints > SS_MAX_JOINTS || (d->n_joints > 0 && !d->joints)) {
    set_error("bad joint table"); return SS_ERR_CONTRACT;
  }
  for (int j = 0; j < d->n_joints; ++j) {
    const SsJointDesc& q = d->joints[j];
    if (q.a < 0 || q.b < 0 || q.a >= d->n_entities || q.b >= d->n_entities || q.a == q.b) {
      set_error("joint " + std::to_string(j) + " has bad entity indices"); return SS_ERR_CONTRACT;
    }
  }
  for (int j = 0; j < d->n_reset_ops; ++j) {
    const SsResetOp& o = d->reset_ops[j];
    const bool uses_entity = o.kind <= SS_RESET_PLACE || o.kind >= SS_RESET_LOADPOS;
    const bool reg_ok = o.r0 >= 0 && o.r0 < SS_RESET_REGS && o.r1 >= 0 && o.r1 < SS_RESET_REGS &&
                        o.r2 >= 0 && o.r2 < SS_RESET_REGS;
    if (o.kind < SS_RESET_SCATTER || o.kind > SS_RESET_ZERO || !reg_ok || (o.axis != 0 && o.axis != 1) ||
        (uses_entity && (o.entity < 0 || o.entity >= d->n_entities))) {
      set_error("bad reset op " + std::to_string(j)); return SS_ERR_CONTRACT;
    }
  }
  return SS_OK;
}

}  // namespace ss

using namespace ss;

extern "C" {

int ss_abi_version(void) { return SS_ABI_VERSION; }

const char* ss_last_error(void) { return g_last_error.c_str(); }

int ss_world_create(const SsWorldDesc* desc, void** out_world) {
  if (!out_world) { set_error("null out pointer"); return SS_ERR_CONTRACT; }
  *out_world = nullptr;
  int rc = validate_desc(desc);
  if (rc) return rc;
  World* w = new (std::nothrow) World();
  if (!w) { set_error("out of host memory"); return SS_ERR_CUDA; }
  w->d = *desc;
  w->ents.assign(desc->entities, desc->entities + desc->n_entities);
  w->pairs.assign(desc->pairs, desc->pairs + desc->n_pairs);
  w->reset_ops.assign(desc->reset_ops, desc->reset_ops + desc->n_reset_ops);
  if (desc->n_joints > 0) w->joints.assign(desc->joints, desc->joints + desc->n_joints);
  w->n_slots = 0;     // draw slots per env: 2 per scatter, 1 per draw
  for (const auto& o : w->reset_ops) w->n_slots += (o.kind == SS_RESET_SCATTER) ? 2 : (o.kind == SS_RESET_DRAW);
  if ((rc = upload(w->ents, &w->d_ents)) || (rc = upload(w->pairs, &w->d_pairs)) ||
      (rc = upload(w->reset_ops, &w->d_reset_ops)) || (rc = upload(w->joints, &w->d_joints))) {
    free_world(w);
    return rc;
  }
  if (desc->lidar_rays > 0) {
    std::vector<double> dirs(desc->lidar_dirs, desc->lidar_dirs + 2 * desc->lidar_rays);
    if ((rc = upload(dirs, &w->d_lidar_dirs))) { free_world(w); return rc; }
  }
  w->scan_cap = (desc->batch + 255) / 256 + 2;
  cudaError_t e = cudaMalloc(reinterpret_cast<void**>(&w->d_scan), w->scan_cap * sizeof(int64_t));
  if (e != cudaSuccess) { free_world(w); return cuda_status(e, "cudaMalloc (scan scratch)"); }
  // the struct copy still points at caller memory; never read those again
  w->d.entities = nullptr;
  w->d.pairs = nullptr;
  w->d.reset_ops = nullptr;
  w->d.lidar_dirs = nullptr;
  w->d.joints = nullptr;
  *out_world = w;
  return SS_OK;
}

int ss_world_destroy(void* world) {
  free_world(static_cast<World*>(world));
  return SS_OK;
}

int ss_env_step(void* world, const SsBuffers* buf, const SsStepIO* io, void* stream) {
  World* w = static_cast<World*>(world);
  if (!w || !buf || !io) { set_error("null argument"); return SS_ERR_CONTRACT; }
  if ((io->mode & SS_DO_PHYSICS) && w->d.n_agents > 0 && !io->actions) {
    set_error("actions required for a physics step"); return SS_ERR_CONTRACT;
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if ((io->mode & SS_DO_PHYSICS) && w->d.n_joints > 0 && w->d.scenario != SS_SCN_PHYSICS_ONLY) {
    set_error("worlds with joints step their physics through ss_world_step (generic kernel)");
    return SS_ERR_CONTRACT;
  }
  switch (w->d.scenario) {
    case SS_SCN_SIMPLE_SPREAD:
    case SS_SCN_TRANSPORT:
    case SS_SCN_FLOCKING:
    case SS_SCN_DROPOUT:
    case SS_SCN_WHEEL:
    case SS_SCN_GIVE_WAY:
    case SS_SCN_PASSAGE:
    case SS_SCN_BALANCE:
    case SS_SCN_WATERFALL:
    case SS_SCN_FOOTBALL:
      return launch_small(*w, buf, io, st);
    case SS_SCN_DISPERSION:
    case SS_SCN_DISCOVERY:
      return launch_large(*w, buf, io, st);
    default:
      return launch_generic(*w, buf, io, nullptr, nullptr, st);
  }
}

int ss_env_rollout(void* world, const SsBuffers* buf, const SsRolloutIO* io, void* stream) {
  World* w = static_cast<World*>(world);
  if (!w || !buf || !io) { set_error("null argument"); return SS_ERR_CONTRACT; }
  if (io->n_steps < 1 || io->n_steps > SS_MAX_ROLLOUT || !io->actions || !io->obs || !io->rew || !io->done) {
    set_error("rollout: 1.." + std::to_string(SS_MAX_ROLLOUT) + " steps with actions and outputs per step");
    return SS_ERR_CONTRACT;
  }
  if (io->check_actions && !io->guard) { set_error("rollout: check_actions needs guard words"); return SS_ERR_CONTRACT; }
  for (int s = 0; s < io->n_steps; ++s) {
    bool ok = io->obs[s] && io->rew[s] && io->done[s];
    for (int i = 0; i < w->d.n_agents; ++i) ok = ok && io->actions[s * w->d.n_agents + i];
    if (!ok) { set_error("rollout: null action or output pointer in step " + std::to_string(s)); return SS_ERR_CONTRACT; }
  }
  return launch_rollout(*w, buf, io, static_cast<cudaStream_t>(stream));
}

int ss_world_step(void* world, const SsBuffers* buf, const float* const* forces,
                  const uint64_t* decode_mask, int32_t count, const int32_t* guard,
                  int32_t guard_count, int32_t* d_status, void* stream) {
  World* w = static_cast<World*>(world);
  if (!w || !buf) { set_error("null argument"); return SS_ERR_CONTRACT; }
  SsStepIO io;
  memset(&io, 0, sizeof(io));
  io.actions = forces;
  io.guard = guard;
  io.guard_count = guard_count;
  io.mode = SS_DO_PHYSICS | (count ? SS_DO_COUNT : 0);
  return launch_generic(*w, buf, &io, decode_mask, d_status, static_cast<cudaStream_t>(stream));
}

int ss_reset(void* world, const SsBuffers* buf, const uint8_t* mask, const int64_t* mask_base,
             const int64_t* mask_total, void* stream) {
  World* w = static_cast<World*>(world);
  if (!w || !buf) { set_error("null argument"); return SS_ERR_CONTRACT; }
  return launch_reset(*w, buf, mask, mask_base, mask_total, static_cast<cudaStream_t>(stream));
}

int ss_mask_count(void* world, const uint8_t* mask, int64_t* count_out, void* stream) {
  World* w = static_cast<World*>(world);
  if (!w || !mask || !count_out) { set_error("null argument"); return SS_ERR_CONTRACT; }
  return launch_mask_count(*w, mask, count_out, static_cast<cudaStream_t>(stream));
}

int ss_check_actions(void* world, const float* const* actions, int32_t* flag_out, void* stream) {
  World* w = static_cast<World*>(world);
  if (!w || !flag_out) { set_error("null argument"); return SS_ERR_CONTRACT; }
  return launch_check_actions(w->d.n_agents, w->d.batch, actions, flag_out,
                              static_cast<cudaStream_t>(stream));
}

int ss_check_action_sets(const float* const* bases, int32_t n_sets, int32_t n_agents, int64_t agent_stride,
                         int64_t n_floats, int32_t* flags, void* stream) {
  if (!bases || !flags || n_sets < 1 || n_sets > SS_MAX_ROLLOUT || n_agents < 1 ||
      (int64_t)n_sets * n_agents > 65535 || n_floats < 0 || agent_stride < n_floats) {
    set_error("check_action_sets: 1.." + std::to_string(SS_MAX_ROLLOUT) + " sets of agent blocks");
    return SS_ERR_CONTRACT;
  }
  for (int s = 0; s < n_sets; ++s)
    if (!bases[s]) { set_error("check_action_sets: null set"); return SS_ERR_CONTRACT; }
  if (n_floats == 0) return cuda_status(cudaMemsetAsync(flags, 0, sizeof(int32_t) * n_sets,
                                                        static_cast<cudaStream_t>(stream)), "flags reset");
  return launch_check_sets(bases, n_sets, n_agents, agent_stride, n_floats, flags,
                           static_cast<cudaStream_t>(stream));
}

int ss_publish_flag(const int32_t* flag, int32_t* host_out, int32_t n, void* stream) {
  if (!flag || !host_out || n < 1 || n > 1024) { set_error("publish_flag: 1..1024 words"); return SS_ERR_CONTRACT; }
  return launch_publish_flag(flag, host_out, n, static_cast<cudaStream_t>(stream));
}

int ss_lidar(void* world, const SsBuffers* buf, int32_t agent, const SsLidarDesc* lidar,
             float* out, void* stream) {
  World* w = static_cast<World*>(world);
  if (!w || !buf || !lidar || !out) { set_error("null argument"); return SS_ERR_CONTRACT; }
  if (agent < 0 || agent >= w->d.n_entities) { set_error("emitter index out of range"); return SS_ERR_CONTRACT; }
  if (lidar->n_rays < 1) { set_error("n_rays must be >= 1"); return SS_ERR_CONTRACT; }
  return launch_lidar(*w, buf, agent, lidar, out, static_cast<cudaStream_t>(stream));
}

int ss_np_trig(const float* x, float* out, int64_t n, int32_t want_cos, void* stream) {
  if ((!x || !out) && n > 0) { set_error("null argument"); return SS_ERR_CONTRACT; }
  return launch_np_trig(x, out, n, want_cos, static_cast<cudaStream_t>(stream));
}

int ss_cast_ray(void* world, const SsBuffers* buf, int32_t exclude, const float* ox,
                const float* oy, const double* angle, double max_range, float* out, void* stream) {
  World* w = static_cast<World*>(world);
  if (!w || !buf || !ox || !oy || !angle || !out) { set_error("null argument"); return SS_ERR_CONTRACT; }
  return launch_cast_ray(*w, buf, exclude, ox, oy, angle, max_range, out,
                         static_cast<cudaStream_t>(stream));
}

int ss_collision_force(const float* pix, const float* piy, const float* pjx, const float* pjy,
                       float d_min, float sign, float contact_ck, float contact_k, float* fx,
                       float* fy, uint8_t* active, int64_t n, void* stream) {
  return launch_collision_force(pix, piy, pjx, pjy, d_min, sign, contact_ck, contact_k, fx, fy,
                                active, n, static_cast<cudaStream_t>(stream));
}

int ss_closest_points(const float* pos_i, const float* rot_i, int32_t shape_i, double dim_i0,
                      double dim_i1, const float* pos_j, const float* rot_j, int32_t shape_j,
                      double dim_j0, double dim_j1, float* out_i, float* out_j, int64_t n,
                      int32_t* d_status, void* stream) {
  ShapeK si, sj;
  si.kind = shape_i; si.d0 = dim_i0; si.d1 = dim_i1;
  sj.kind = shape_j; sj.d0 = dim_j0; sj.d1 = dim_j1;
  if (shape_i < SS_SPHERE || shape_i > SS_LINE || shape_j < SS_SPHERE || shape_j > SS_LINE) {
    set_error("unsupported shape pair");
    return SS_ERR_SHAPE_PAIR;
  }
  return launch_closest_points(pos_i, rot_i, si, pos_j, rot_j, sj, out_i, out_j, n, d_status,
                               static_cast<cudaStream_t>(stream));
}

}  // extern "C"
