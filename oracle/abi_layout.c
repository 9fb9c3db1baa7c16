/* abi_layout — prints sizeof/offsetof of every C-ABI struct as JSON so the
 * ctypes mirror (paper_2207_03530_b200/_native.py) can be checked against
 * the header as the C compiler lays it out.  TEST INFRASTRUCTURE. */
#include <stddef.h>
#include <stdio.h>

#include "../include/swarmsim_b200.h"

#define F(S, m) printf("\"%s.%s\": %zu, ", #S, #m, offsetof(S, m))
#define Z(S) printf("\"%s\": %zu, ", #S, sizeof(S))

int main(void) {
  printf("{");
  Z(SsEntityDesc); F(SsEntityDesc, shape); F(SsEntityDesc, slot); F(SsEntityDesc, dim0);
  F(SsEntityDesc, dim1); F(SsEntityDesc, inv_m_dt); F(SsEntityDesc, u_mult);
  Z(SsPairDesc); F(SsPairDesc, d_min); F(SsPairDesc, sign); F(SsPairDesc, d2_act);
  Z(SsResetOp); F(SsResetOp, lo_x); F(SsResetOp, range_y); F(SsResetOp, r0); F(SsResetOp, axis);
  Z(SsWorldDesc); F(SsWorldDesc, batch); F(SsWorldDesc, max_steps); F(SsWorldDesc, dt);
  F(SsWorldDesc, entities); F(SsWorldDesc, pairs); F(SsWorldDesc, reset_ops); F(SsWorldDesc, sc);
  F(SsWorldDesc, sd); F(SsWorldDesc, si); F(SsWorldDesc, lidar_rays); F(SsWorldDesc, lidar_max_range);
  F(SsWorldDesc, lidar_dirs); F(SsWorldDesc, substeps); F(SsWorldDesc, n_joints); F(SsWorldDesc, joints);
  Z(SsJointDesc); F(SsJointDesc, ox_a); F(SsJointDesc, dist); F(SsJointDesc, stiffness); F(SsJointDesc, rotate_b);
  Z(SsBuffers); F(SsBuffers, rng); F(SsBuffers, rng_cur);
  Z(SsStepIO); F(SsStepIO, obs_agent_stride); F(SsStepIO, mode); F(SsStepIO, guard); F(SsStepIO, raw_forces);
  F(SsStepIO, guard_count);
  Z(SsRolloutIO); F(SsRolloutIO, actions); F(SsRolloutIO, obs_agent_stride); F(SsRolloutIO, guard); F(SsRolloutIO, check_actions);
  Z(SsLidarDesc); F(SsLidarDesc, max_range); F(SsLidarDesc, dir_table);
  printf("\"end\": 0}\n");
  return 0;
}
