/* swarmsim_b200.h — C-ABI of the B200 batched environment step.
 *
 * The reference (swarmsim 0.1.0, pure Python + numpy) has no FFI; its hot
 * path is the Python call chain
 *     Env.step            /root/reference/pkg/src/swarmsim/env.py:209-235
 *       decode_action     env.py:71-145
 *       world_step        dynamics.py:123-184   (+ closest_points geometry.py:120,
 *                                                collision_force dynamics.py:36,
 *                                                integrate dynamics.py:69)
 *       Scenario.post_step / reward / done / observation   env.py:227-233
 *     Env.reset           env.py:189-198 -> Scenario.reset_world_at
 *     lidar_scan          sensors.py:138-146
 * Every entry point below replaces one of those seams with a stream-ordered
 * launch.  All buffer pointers are DEVICE memory owned by the caller (the
 * Python host side allocates them as torch tensors); the library borrows
 * them for the duration of the call and never allocates inside a step.
 * Only SsWorld (the static scene descriptor, the analog of the pair cache at
 * core.py:247-251) is owned by the library.
 *
 * Return value: 0 on success, a negative SsStatus otherwise; the message is
 * available from ss_last_error() (thread-local).
 */
#ifndef SWARMSIM_B200_H
#define SWARMSIM_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SS_ABI_VERSION 2
#define SS_RNG_WORDS 12          /* counter[4] key[2] buffer[4] buffer_pos spare */
#define SS_MAX_ENTITIES 1024
#define SS_MAX_AGENTS 256
#define SS_MAX_RESET_OPS 1024
#define SS_MAX_JOINTS 1024
#define SS_MAX_SUBSTEPS 1024

typedef enum SsStatus {
  SS_OK = 0,
  SS_ERR_CONTRACT = -1,        /* -> ContractViolation   (errors.py:8)  */
  SS_ERR_SHAPE_PAIR = -2,      /* -> UnsupportedShapePair (errors.py:12) */
  SS_ERR_SCENARIO = -3,        /* -> UnknownScenario      (errors.py:16) */
  SS_ERR_CUDA = -4,            /* CUDA launch / runtime failure          */
  SS_ERR_UNSUPPORTED = -5      /* size not instantiated for a fused kernel */
} SsStatus;

typedef enum SsShape { SS_SPHERE = 0, SS_BOX = 1, SS_LINE = 2 } SsShape;

typedef enum SsScenario {
  SS_SCN_PHYSICS_ONLY = 0,     /* world_step only; reward/obs by Python hooks */
  SS_SCN_SIMPLE_SPREAD = 1,    /* scenarios/simple_spread.py */
  SS_SCN_TRANSPORT = 2,        /* scenarios/transport.py     */
  SS_SCN_FLOCKING = 3,         /* scenarios/flocking.py (+ optional Lidar obs) */
  SS_SCN_DISPERSION = 4,       /* scenarios/dispersion.py    */
  SS_SCN_DISCOVERY = 5,        /* scenarios/discovery.py     */
  SS_SCN_DROPOUT = 6,          /* scenarios/dropout.py (catalog); flags[0..1] = float64 energy spent */
  SS_SCN_WHEEL = 7,            /* scenarios/wheel.py (catalog): reward/obs kernel; physics by world_step */
  SS_SCN_GIVE_WAY = 8,         /* scenarios/give_way.py (catalog): reward/obs kernel; physics by world_step */
  SS_SCN_PASSAGE = 9,          /* scenarios/passage.py (catalog): reward/obs kernel; physics by world_step */
  SS_SCN_BALANCE = 10,         /* scenarios/balance.py (catalog): reward/obs kernel; physics by world_step */
  SS_SCN_WATERFALL = 11,       /* scenarios/waterfall.py (catalog): reward/obs kernel; physics by world_step */
  SS_SCN_FOOTBALL = 12         /* scenarios/football.py (catalog): reward/obs kernel; physics by world_step */
} SsScenario;

/* Step phases (bit flags of SsStepIO.mode). A full Env.step is SS_MODE_STEP. */
enum {
  SS_DO_PHYSICS = 1,   /* decode + world_step                  env.py:218-226 */
  SS_DO_POST = 2,      /* scenario.post_step                   env.py:227     */
  SS_DO_COUNT = 4,     /* step_count += 1                      env.py:228     */
  SS_DO_REWARD = 8,    /* rewards                              env.py:229-231 */
  SS_DO_DONE = 16,     /* dones = done | step_count>=max_steps  env.py:232     */
  SS_DO_OBS = 32,      /* observations                         env.py:233     */
  SS_MODE_STEP = 63
};

/* Per-entity static descriptor (core.py:120-198, shapes.py:15-73). Float
 * fields are pre-rounded on the host exactly as numpy rounds them. */
typedef struct SsEntityDesc {
  int32_t shape;          /* SsShape */
  int32_t movable, rotatable, collidable;
  int32_t is_agent;
  int32_t slot;           /* movable: row of dyn[]; else row of stat[]        */
  double dim0, dim1;      /* sphere radius | box length,width | line length (python floats) */
  float inv_m_dt;         /* f32(f32(1/mass) * f32(dt))     dynamics.py:78   */
  float inv_i_dt;         /* f32(f32(1/moi)  * f32(dt))     dynamics.py:84   */
  float max_speed;        /* f32(max_speed); <= 0 means None                  */
  float grav_x, grav_y;   /* f32(g) * f32(mass)             dynamics.py:154  */
  float u_range;          /* agents: clip bound            env.py:97         */
  float u_mult;           /* agents: f32(u_multiplier)                        */
} SsEntityDesc;

/* One collidable pair (i < j) of the static pair list (dynamics.py:89-100). */
typedef struct SsPairDesc {
  int32_t i, j;
  float d_min;            /* f32(min_contact_distance)      shapes.py:65     */
  float sign;             /* +1 if (i+j) even else -1       dynamics.py:169  */
  float d2_act;           /* largest f32 x with fl(sqrt(x)) <= d_min: the pair is
                             active iff x*x+y*y <= d2_act (no sqrt needed)     */
} SsPairDesc;

/* The reset program: one instruction per reference reset action, in the
 * scenario's call order (reset_world_at: common.py:11-34 scatter / place,
 * plus the catalog tasks' relative placements and angle draws).  Per env it
 * runs on a float32 register file R[SS_RESET_REGS]: the reference's draws
 * are float32 (SeededRng.uniform casts, batching.py:185-186) and Python-float
 * operands meeting them stay float32 (NEP 50), so every value a reset program
 * combines is a float32.  Every draw instruction takes the next draw slot
 * (x before y), so a whole-batch reset reads draw slot*Bg + e and the env of
 * rank r in a masked reset reads r*n_slots + slot (= sequential
 * reset(env_index=i) calls in ascending i). */
typedef enum SsResetKind {
  SS_RESET_SCATTER = 0,   /* pos = f32(lo + range * u) per axis (2 slots); zero motion      */
  SS_RESET_PLACE = 1,     /* pos = (f32(lo_x), f32(lo_y)); zero motion                      */
  SS_RESET_DRAW = 2,      /* R[r0] = f32(lo_x + range_x * u)               (1 slot)         */
  SS_RESET_CONST = 3,     /* R[r0] = f32(lo_x)                                              */
  SS_RESET_ADD = 4,       /* R[r0] = R[r1] + R[r2]   (float32)                              */
  SS_RESET_NEG = 5,       /* R[r0] = -R[r1]                                                 */
  SS_RESET_LOADPOS = 6,   /* R[r0] = pos[entity][axis]                                      */
  SS_RESET_SETPOS = 7,    /* pos[entity] = (R[r0], R[r1]); velocity kept                     */
  SS_RESET_SETROT = 8,    /* rot[entity] = R[r0]                                            */
  SS_RESET_ZERO = 9       /* zero_motion: vel = 0, ang_vel = 0 (core.py:94-103)              */
} SsResetKind;
#define SS_RESET_REGS 16

typedef struct SsResetOp {
  int32_t entity;         /* entity index (-1 for register-only instructions) */
  int32_t kind;           /* SsResetKind */
  double lo_x, lo_y;      /* scatter: lower corner | place: x, y | draw: low | const: value */
  double range_x, range_y;/* scatter / draw: hi - lo (float64, as numpy computes) */
  int32_t r0, r1, r2;     /* register operands */
  int32_t axis;           /* loadpos: 0 = x, 1 = y */
} SsResetOp;

/* Distance joint (extension; the reference has none — SPEC.md:204 lists
 * joints as a non-goal).  VMAS-style penalty constraint between anchor points
 * of entities a and b: anchor = pos + R(rot) * (ox, oy) (body-frame offsets,
 * float32).  With delta = anchor_a - anchor_b and dist = |delta|, a pair of
 * softplus penalties keeps dist at `dist`: repulsive when dist < target,
 * attractive when dist > target, none when dist < 1e-6 or dist == target.
 *   z   = |target - dist| / k,   pen = softplus(z) * k   (k = contact_margin)
 *   f_a = s * stiffness * (delta / dist) * pen,  s = +1 repulsive, -1 attractive
 *   f_b = -f_a; torques r x f on rotatable ends when rotate_a / rotate_b.
 * Joint forces are added after every pair contact, in joint-list order. */
typedef struct SsJointDesc {
  int32_t a, b;           /* entity indices (a != b)                          */
  float ox_a, oy_a;       /* anchor offset on a, body frame (f32)             */
  float ox_b, oy_b;       /* anchor offset on b, body frame (f32)             */
  float dist;             /* f32 target distance between the anchors          */
  float stiffness;        /* f32 force multiplier                             */
  int32_t rotate_a, rotate_b;  /* apply the joint torque to a / b             */
} SsJointDesc;

typedef struct SsWorldDesc {
  int32_t abi_version;    /* SS_ABI_VERSION */
  int32_t scenario;       /* SsScenario */
  int32_t n_entities;     /* agents first (core.py:237-242) */
  int32_t n_agents;
  int32_t n_dyn, n_stat;  /* rows of the dyn / stat state buffers */
  int32_t obs_dim;        /* per-agent observation width */
  int32_t n_flag_words;   /* uint32 rows of SsBuffers.flags */
  int64_t batch;          /* envs held by this process (shard) */
  int64_t env_offset;     /* global index of local env 0 */
  int64_t global_batch;   /* envs across all shards (RNG stream layout) */
  int64_t max_steps;
  float dt;               /* f32(dt) */
  float keep;             /* f32(1 - damping) */
  float contact_ck;       /* f32(contact_force * contact_margin) */
  float contact_k;        /* f32(contact_margin) */
  int32_t has_gravity;
  int32_t n_pairs;
  const SsEntityDesc* entities;
  const SsPairDesc* pairs;
  int32_t n_reset_ops;
  const SsResetOp* reset_ops;
  float sc[16];           /* scenario float32 constants */
  double sd[8];           /* scenario float64 constants */
  int32_t si[8];          /* scenario int constants */
  /* optional Lidar appended to each agent's observation (flocking config) */
  int32_t lidar_rays;     /* 0 = none */
  int32_t lidar_attach_rotation;
  double lidar_max_range;
  double lidar_start, lidar_span;
  const double* lidar_dirs;   /* HOST [lidar_rays][2]: numpy cos/sin of the rot=0 angles */
  /* ABI 2 extensions (both default to the reference's behaviour) */
  int32_t substeps;       /* physics sub-steps per Env.step (>= 1; 1 = reference).
                             dt, inv_m_dt, inv_i_dt are already the SUB-step
                             values f32(dt / substeps); keep stays f32(1 - damping)
                             per sub-step (VMAS semantics). Actions, scripts,
                             post_step, rewards, dones and observations run once. */
  int32_t n_joints;       /* 0 = none (reference); worlds with joints run the
                             generic physics kernel */
  const SsJointDesc* joints;
} SsWorldDesc;

/* Device state, all row-major [row][B][...], env index contiguous. */
typedef struct SsBuffers {
  float* dyn;             /* [n_dyn][B][4]  px py vx vy of movable entities */
  float* stat;            /* [n_stat][B][2] position of non-movable entities */
  float* stat_vel;        /* [n_stat][B][2] velocity of non-movable entities */
  float* rot;             /* [n_entities][B][2] rot, ang_vel */
  int64_t* step_count;    /* [B] */
  uint32_t* flags;        /* [n_flag_words][B] scenario bit flags */
  float* aux;             /* [B] scenario scalar (dispersion fresh_bites) */
  uint64_t* rng;          /* [2][SS_RNG_WORDS] double-buffered Philox state */
  int32_t rng_cur;        /* which half of rng[] is current (input) */
} SsBuffers;

typedef struct SsStepIO {
  const float* const* actions; /* HOST array of n_agents device pointers, each [B][2] f32 */
  float* obs;             /* obs of agent a, env e at obs[a*obs_agent_stride + e*obs_dim] */
  int64_t obs_agent_stride;
  float* rew;             /* [n_agents][B] */
  uint8_t* done;          /* [B] */
  int32_t mode;           /* SS_DO_* flags */
  const int32_t* guard;   /* optional device flags: if any of guard[0 .. guard_count) is
                             nonzero the launch is a no-op (the NaN verdict, env.py:85) */
  int32_t raw_forces;     /* nonzero: actions are final forces (discrete / noisy /
                             scripted agents decoded by the host); skip decode_action */
  int32_t guard_count;    /* words at guard (0 means 1) */
} SsStepIO;

/* An open-loop rollout of n_steps consecutive Env.steps in ONE launch
 * (extension): the step kernels' work with each env's state kept on chip
 * between the steps — it is read once before the first and written once
 * after the last, so a step moves only its actions and outputs.  Results are
 * bitwise those of n_steps ss_env_step calls (SS_MODE_STEP).  Scenarios
 * without a rollout kernel return SS_ERR_UNSUPPORTED (take the per-step
 * path).  guard (device, may be NULL): n_steps NaN words; step s runs only
 * while words 0..s are all zero, so a NaN in step k's actions leaves the
 * state as after step k-1.  check_actions (guard required): the call itself
 * zeroes guard and fills guard[s] with the NaN verdict of step s's actions
 * (env.py:85) in ONE scan launch over all the steps, before the rollout. */
#define SS_MAX_ROLLOUT 16
typedef struct SsRolloutIO {
  int32_t n_steps;                 /* 1 .. SS_MAX_ROLLOUT */
  const float* const* actions;     /* HOST [n_steps * n_agents] device pointers, each [B][2] f32 */
  float* const* obs;               /* HOST [n_steps] device pointers, layout of SsStepIO.obs */
  int64_t obs_agent_stride;
  float* const* rew;               /* HOST [n_steps] device pointers, each [n_agents][B] */
  uint8_t* const* done;            /* HOST [n_steps] device pointers, each [B] */
  int32_t* guard;                  /* device [n_steps] or NULL */
  int32_t check_actions;           /* nonzero: scan the actions into guard first */
} SsRolloutIO;

typedef struct SsLidarDesc {
  int32_t n_rays;
  double max_range;       /* compared/returned as in sensors.py:135 */
  double start_angle, span;  /* ray m: start + m*span/n_rays (+ rot) */
  int32_t attach_rotation;
  const double* dir_table;   /* optional device [n_rays][2] cos/sin for rot == 0 */
} SsLidarDesc;

int ss_abi_version(void);
const char* ss_last_error(void);

/* Build / free the static scene descriptor (pair list, constants, reset
 * program) for one World.  Replaces the Python pair cache core.py:247-251. */
int ss_world_create(const SsWorldDesc* desc, void** out_world);
int ss_world_destroy(void* world);

/* One fused Env.step for every env (env.py:209-235).  For scenario
 * SS_SCN_PHYSICS_ONLY only SS_DO_PHYSICS|SS_DO_COUNT apply (world_step,
 * dynamics.py:123-184). */
int ss_env_step(void* world, const SsBuffers* buf, const SsStepIO* io, void* stream);

/* n_steps fused steps in one launch (SsRolloutIO): simple_spread,
 * transport / reverse_transport and flocking (1..8 agents) without
 * sub-steps or joints; SS_ERR_UNSUPPORTED otherwise, SS_ERR_CONTRACT for a
 * bad step count or a null pointer (nothing launched). */
int ss_env_rollout(void* world, const SsBuffers* buf, const SsRolloutIO* io, void* stream);

/* Env.reset (env.py:189-198) -> Scenario.reset_world_at.  mask == NULL
 * resets every env with the reference's whole-batch draw order (x block then
 * y block per scatter, batching.py:212-213); otherwise mask[B] (uint8) resets
 * the selected envs exactly as sequential reset(env_index=i) calls in
 * ascending i.  `mask_base` (device, may be NULL) is the number of selected
 * envs on lower shards and `mask_total` (device, may be NULL) the selected
 * count over all shards; both NULL means unsharded.  Advances buf->rng into
 * the other half; the caller flips rng_cur afterwards. */
int ss_reset(void* world, const SsBuffers* buf, const uint8_t* mask,
             const int64_t* mask_base, const int64_t* mask_total, void* stream);

/* Count of selected envs in mask[B] into *count_out (device int64). */
int ss_mask_count(void* world, const uint8_t* mask, int64_t* count_out, void* stream);

/* NaN scan of the actions (env.py:85, dynamics.py:112): sets *flag_out
 * (device int32) to nonzero when any value is NaN.  Does not clear it. */
int ss_check_actions(void* world, const float* const* actions, int32_t* flag_out, void* stream);

/* NaN scans of n_sets action sets in ONE launch (extension; a replay of
 * n_sets steps): set s holds n_agents blocks of n_floats f32, agent_stride
 * floats apart, from device pointer bases[s] (HOST array).  Zeroes
 * flags[0 .. n_sets) and sets flags[s] nonzero when set s holds a NaN
 * (env.py:85 per step).  1 <= n_sets <= SS_MAX_ROLLOUT. */
int ss_check_action_sets(const float* const* bases, int32_t n_sets, int32_t n_agents, int64_t agent_stride,
                         int64_t n_floats, int32_t* flags, void* stream);

/* Publish the NaN verdict to the host (extension): host_out[i] = flag[i]
 * for i < n, stored by a one-CTA kernel into host-mapped pinned memory
 * (cudaHostAlloc; unified addressing), so the caller waits on an event
 * instead of a device-to-host copy that would queue behind observation
 * copies in flight on the copy engine (Env.step(validate=True)). */
int ss_publish_flag(const int32_t* flag, int32_t* host_out, int32_t n, void* stream);

/* lidar_scan (sensors.py:138-146) for one agent: out[B][n_rays] f32. */
int ss_lidar(void* world, const SsBuffers* buf, int32_t agent, const SsLidarDesc* lidar,
             float* out, void* stream);

/* cast_ray (sensors.py:113-135): out[e] = nearest hit from (ox[e], oy[e])
 * along angle[e] (float64), skipping entity `exclude` (-1: none). */
int ss_cast_ray(void* world, const SsBuffers* buf, int32_t exclude, const float* ox,
                const float* oy, const double* angle, double max_range, float* out, void* stream);

/* np.cos (want_cos != 0) / np.sin of a float32 array, bit-exact with numpy's
 * float32 loops (used by the scenario observations of wheel.py:72-73,
 * balance.py obs, and by Vec2.rotated, batching.py:132-134). */
int ss_np_trig(const float* x, float* out, int64_t n, int32_t want_cos, void* stream);

/* Function-level seams used by the reference's unit tests. All arrays [n]. */
/* collision_force (dynamics.py:36-66): force on i and the active mask. */
int ss_collision_force(const float* pix, const float* piy, const float* pjx, const float* pjy,
                       float d_min, float sign, float contact_ck, float contact_k,
                       float* fx, float* fy, uint8_t* active, int64_t n, void* stream);
/* closest_points (geometry.py:120-163) between two posed shapes.  Shape
 * dimensions are the Python floats of shapes.py.  *d_status (device int32)
 * is set nonzero on an unsupported pair. */
int ss_closest_points(const float* pos_i /*[n][2]*/, const float* rot_i, int32_t shape_i,
                      double dim_i0, double dim_i1,
                      const float* pos_j /*[n][2]*/, const float* rot_j, int32_t shape_j,
                      double dim_j0, double dim_j1,
                      float* out_i /*[n][2]*/, float* out_j /*[n][2]*/, int64_t n,
                      int32_t* d_status, void* stream);

/* Module-level world_step(world, actions) (dynamics.py:123-184) for any
 * world: forces[a] is agent a's force [B][2] (device); decode_mask bit a
 * (4 x uint64, NULL = all) applies decode_action's clip*u_multiplier to it
 * (Env.step path) instead of using it as-is (AgentAction / action_script
 * path).  count != 0 also increments step_count.  guard (device, may be
 * NULL): if any of guard[0 .. guard_count) is nonzero the launch leaves every
 * buffer untouched (the NaN verdict of ss_check_actions, env.py:85).
 * *d_status as above. */
int ss_world_step(void* world, const SsBuffers* buf, const float* const* forces,
                  const uint64_t* decode_mask, int32_t count, const int32_t* guard,
                  int32_t guard_count, int32_t* d_status, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* SWARMSIM_B200_H */
