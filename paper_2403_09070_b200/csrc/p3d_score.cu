// Solution score (evaluate_score, model.py:364-400): the
// die-to-die HPWL of a placed solution, net-parallel.  Per net: each pin at
// its instance's lower-left corner + rotated half size + rotated offset of
// the instance's die (solution_pin_xy, model.py:352-361), extents per die,
// the HBT centre joining both partial nets; crossing / HBT consistency flags
// for the caller's SolutionError.  Compiled -fmad=false (Python float order).
#include <math.h>

#include "p3d_common.cuh"
#include "p3d_internal.cuh"

namespace p3d {

namespace {

__device__ __forceinline__ void turn(double ox, double oy, int q, double& rx, double& ry) {
  switch (q & 3) {  // model.py:278-289
    case 0: rx = ox; ry = oy; break;
    case 1: rx = -oy; ry = ox; break;
    case 2: rx = -ox; ry = -oy; break;
    default: rx = oy; ry = -ox; break;
  }
}

__global__ void __launch_bounds__(256) score_kernel(ScoreArgs a) {
  __shared__ double red[32 * 2];
  double acc[2] = {0.0, 0.0};  // hpwl, hbt count
  int bad = 0;
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < a.n_net; j += gridDim.x * blockDim.x) {
    double lo[2][2] = {{P3D_INF, P3D_INF}, {P3D_INF, P3D_INF}};
    double hi[2][2] = {{-P3D_INF, -P3D_INF}, {-P3D_INF, -P3D_INF}};
    int cnt[2] = {0, 0};
    for (int k = a.net_ptr[j]; k < a.net_ptr[j + 1]; ++k) {
      const int i = a.pin_inst[k];
      const int d = a.die[i] ? 1 : 0, q = (int)(a.rot[i] & 3);
      const double w0 = d ? a.w_top[i] : a.w_bot[i], h0 = d ? a.h_top[i] : a.h_bot[i];
      const double w = (q & 1) ? h0 : w0, h = (q & 1) ? w0 : h0;
      double rx, ry;
      turn(d ? a.ox_top[k] : a.ox_bot[k], d ? a.oy_top[k] : a.oy_bot[k], q, rx, ry);
      const double px = a.x[i] + w / 2 + rx, py = a.y[i] + h / 2 + ry;
      lo[d][0] = fmin(lo[d][0], px); hi[d][0] = fmax(hi[d][0], px);
      lo[d][1] = fmin(lo[d][1], py); hi[d][1] = fmax(hi[d][1], py);
      cnt[d] += 1;
    }
    const bool crossing = cnt[0] > 0 && cnt[1] > 0;
    const bool has = a.hbt_ok[j] != 0;
    if (crossing != has) bad += 1;
    if (has) {
      acc[1] += 1.0;
      const double cx = a.hbt_x[j] + a.half, cy = a.hbt_y[j] + a.half;
      for (int d = 0; d < 2; ++d)
        if (crossing || cnt[d]) {
          lo[d][0] = fmin(lo[d][0], cx); hi[d][0] = fmax(hi[d][0], cx);
          lo[d][1] = fmin(lo[d][1], cy); hi[d][1] = fmax(hi[d][1], cy);
          cnt[d] += 1;
        }
    }
    for (int d = 0; d < 2; ++d)
      if (cnt[d]) acc[0] += hi[d][0] - lo[d][0] + hi[d][1] - lo[d][1];
  }
  if (bad) atomicAdd(a.n_bad, bad);
  block_sum<2>(acc, red);
  if (threadIdx.x == 0) {
    a.partials[blockIdx.x] = acc[0];
    a.partials[gridDim.x + blockIdx.x] = acc[1];
  }
  if (last_block(a.counter)) {
    const double h = ordered_sum(a.partials, gridDim.x, red);
    const double c = ordered_sum(a.partials + gridDim.x, gridDim.x, red);
    if (threadIdx.x == 0) {
      a.out[0] = h;
      a.out[1] = c;
      a.out[2] = h + a.cost * c;
    }
  }
}

}  // namespace

void launch_score(const ScoreArgs& a, cudaStream_t s) {
  score_kernel<<<grid_blocks(a.n_net, 256, 1024), 256, 0, s>>>(a);
}

}  // namespace p3d
