// k2_common.cuh -- K2's launch arguments and the device error record.
#pragma once
#include <cuda_runtime.h>

#include "decide.cuh"

namespace es {

struct ReplayArgs {  // one es_replay_traces call
  int64_t n_scen;
  const uint16_t *cfg_idx;
  const uint64_t *arr_off;
  const uint32_t *arrival;
  uint32_t *completion;
  uint8_t *exit_used;
  uint32_t *lat;
  uint64_t *stats;
  int64_t dec_cap;
  uint32_t *dec_t;
  uint8_t *dec_m, *dec_e;
  uint16_t *dec_B;
  uint32_t *dec_L;
  uint64_t *dec_S;
  uint8_t *dec_f;
  DevStatus *dstat;
  unsigned long long *work;
  const uint32_t *order;  // scenario hand-out order (longest traces first), or null
  uint32_t stage_bytes;   // image bytes staged in shared memory (core only: H read from global)
  bool any_simple;  // some cfg selects by LQF / EDF / deferred batching (Q26, Q27)
  bool any_score;   // some cfg selects by the stability score (Eq. 7)
  bool any_grid;    // some cfg scores every (m, e, b) cell (f2, Q28)
};

__device__ __forceinline__ void report(DevStatus *ds, uint32_t code, int64_t item) {
  if (atomicCAS(&ds->code, 0u, code) == 0u) ds->item = (unsigned long long)item;
}

}  // namespace es
