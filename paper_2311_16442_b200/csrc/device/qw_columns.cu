// qw_columns.cu -- small batches (2..16 columns) on the batch-1 kernels.
//
// The reference computes a batch as independent GEMVs (one matvec per
// activation, engine.cpp:169-249).  Running the batch-1 kernel once per
// column pays the per-launch cost b times; K4 (qw_gemm.cu) pays ~7 us of
// fixed cost.  Here up to kMaxSeg (8) columns share ONE launch: the grid is split
// over the columns exactly like a layer group (qw_gemv.cu / qw_mma.cu group
// launches), every segment the same layer with its own x and y.  The
// segments' CTAs stream the same records at the same time, so HBM delivers
// the weights about once and L2 serves the other columns; the per-launch
// costs (dependency release, first weights, tail) are paid once per launch.
#include <cuda_runtime.h>

#include <algorithm>

#include "qw_device.hpp"

namespace qwdev {

int plan_columns(DeviceLayer& L, int num_sms, const uint32_t* host_row_ptr) {
  const DeviceLayer* same[kMaxSeg];
  const uint32_t* rps[kMaxSeg];
  std::fill(same, same + kMaxSeg, &L);
  std::fill(rps, rps + kMaxSeg, host_row_ptr);
  for (uint32_t n = 2; n <= kMaxSeg; ++n) {
    GemvPlan& p = L.cplan[n - 2];
    if (plan_gemv_group(p, same, rps, n, num_sms)) p = GemvPlan{}, p.grid = 0;  // per-column fallback
    MmaPlan& m = L.mcplan[n - 2];
    m = MmaPlan{};
    if (L.mrecs && plan_mma(m, same, rps, n, num_sms)) m = MmaPlan{}, m.grid = 0;
  }
  return 0;
}

int launch_columns(const DeviceLayer& L, const float* x, uint32_t batch, float* y, void* stream, bool pdl,
                   uint32_t flags) {
  const DeviceLayer* same[kMaxSeg];
  std::fill(same, same + kMaxSeg, &L);
  for (uint32_t c0 = 0; c0 < batch;) {
    const uint32_t n = std::min<uint32_t>(kMaxSeg, batch - c0);
    const float* xs[kMaxSeg];
    float* ys[kMaxSeg];
    for (uint32_t s = 0; s < n; ++s) xs[s] = x + (size_t)(c0 + s) * L.g.cols, ys[s] = y + (size_t)(c0 + s) * L.g.rows;
    int e = 0;
    if (L.mrecs) {
      const MmaPlan* p = n == 1 ? &L.mplan : &L.mcplan[n - 2];
      if (n > 1 && p->grid == 0) {  // no column plan: one launch per column
        for (uint32_t s = 0; s < n && !e; ++s)
          e = launch_mma(L.mplan, same, 1, xs + s, ys + s, stream, pdl, flags, nullptr);
      } else {
        uint32_t slots[kMaxSeg];
        for (uint32_t s = 0; s < kMaxSeg; ++s) slots[s] = s;
        e = launch_mma(*p, same, n, xs, ys, stream, pdl, flags, slots);
      }
    } else {
      const GemvPlan* p = n == 1 ? &L.plan : &L.cplan[n - 2];
      if (n > 1 && p->grid == 0) {
        for (uint32_t s = 0; s < n && !e; ++s)
          e = launch_gemv_group(L.plan, same, 1, xs + s, ys + s, stream, pdl, flags, nullptr, 1, false);
      } else {
        e = launch_gemv_group(*p, same, n, xs, ys, stream, pdl, flags, nullptr, 1, false);
      }
    }
    if (e) return e;
    c0 += n;
  }
  return 0;
}

// launches of one launch_columns call
uint32_t column_launches(const DeviceLayer& L, uint32_t batch) {
  uint32_t total = 0;
  for (uint32_t c0 = 0; c0 < batch;) {
    const uint32_t n = std::min<uint32_t>(kMaxSeg, batch - c0);
    const bool planned = n == 1 || (L.mrecs ? L.mcplan[n - 2].grid : L.cplan[n - 2].grid) != 0;
    total += planned ? 1 : n;
    c0 += n;
  }
  return total;
}

}  // namespace qwdev
