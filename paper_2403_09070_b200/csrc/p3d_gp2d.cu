// Multi-die 2D GP (run_gp2d_multi, gp.py:531-690): the
// partial-net weighted-average wirelength over the augmented pin list (each
// HBT joins both partial nets of its crossing net, gp.py:482-498) and its
// per-object owner sums.  Compiled with -fmad=false and written in numpy's
// operation order (wirelength.py:76-98) so values and gradients round like
// the reference's _segment_wa (exp itself is CUDA's correctly-rounded-to-1-ulp
// exp, numpy's is SVML/glibc: <= 1 ulp apart).
#include <math.h>

#include "p3d_common.cuh"
#include "p3d_internal.cuh"

namespace p3d {

namespace {

struct Seg {
  double hi, lo, s1p, sxp, s1m, sxm, vp, vm;
};

// one (net, die) segment on one axis: extrema, sums in pin order
__device__ __forceinline__ void seg_stats(const Gp2dWlArgs& a, int b, int e, int die, int axis,
                                          double gamma, Seg& s) {
  s.hi = -P3D_INF;
  s.lo = P3D_INF;
  for (int k = b; k < e; ++k) {
    if (a.pin_top[k] != die) continue;
    const double v = a.pos[(long long)axis * a.n_obj + a.pin_obj[k]] + (axis ? a.pin_oy[k] : a.pin_ox[k]);
    s.hi = fmax(s.hi, v);
    s.lo = fmin(s.lo, v);
  }
  s.s1p = s.sxp = s.s1m = s.sxm = 0.0;
  for (int k = b; k < e; ++k) {
    if (a.pin_top[k] != die) continue;
    const double v = a.pos[(long long)axis * a.n_obj + a.pin_obj[k]] + (axis ? a.pin_oy[k] : a.pin_ox[k]);
    const double ep = exp((v - s.hi) / gamma), em = exp((s.lo - v) / gamma);
    s.s1p += ep;
    s.sxp += v * ep;
    s.s1m += em;
    s.sxm += v * em;
  }
  const bool live = s.s1p > 0;
  s.vp = live ? s.sxp / s.s1p : 0.0;
  s.vm = live ? s.sxm / s.s1m : 0.0;
}

__global__ void __launch_bounds__(256) gp2d_wl_kernel(Gp2dWlArgs a) {
  __shared__ double red[32];
  double acc[1] = {0.0};
  const double gamma = a.gamma;
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < a.n_net; j += gridDim.x * blockDim.x) {
    const int b = a.net_ptr[j], e = a.net_ptr[j + 1];
    for (int axis = 0; axis < 2; ++axis) {
      Seg sg[2];
      for (int die = 0; die < 2; ++die) {
        seg_stats(a, b, e, die, axis, gamma, sg[die]);
        acc[0] += sg[die].s1p > 0 ? sg[die].vp - sg[die].vm : 0.0;
      }
      for (int k = b; k < e; ++k) {  // wirelength.py:94-96
        const Seg& s = sg[a.pin_top[k]];
        const double v = a.pos[(long long)axis * a.n_obj + a.pin_obj[k]] + (axis ? a.pin_oy[k] : a.pin_ox[k]);
        const double ep = exp((v - s.hi) / gamma), em = exp((s.lo - v) / gamma);
        const double g = ep / s.s1p * (1 + (v - s.vp) / gamma) - em / s.s1m * (1 - (v - s.vm) / gamma);
        a.rec[2 * (long long)a.pin_slot[k] + axis] = g;
      }
    }
  }
  block_sum<1>(acc, red);
  if (threadIdx.x == 0) a.partials[blockIdx.x] = acc[0];
  if (last_block(a.counter)) {
    const double s = ordered_sum(a.partials, gridDim.x, red);
    if (threadIdx.x == 0) *a.value = s;
  }
}

// owner sums in pin order (np.bincount(pin_obj, g)): out [n_obj][2]
__global__ void __launch_bounds__(256) gp2d_gather_kernel(int n_obj, const int32_t* obj_slot_ptr,
                                                         const double* rec, double* out) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n_obj; i += gridDim.x * blockDim.x) {
    double sx = 0.0, sy = 0.0;
    for (int s = obj_slot_ptr[i]; s < obj_slot_ptr[i + 1]; ++s) {
      sx += rec[2 * (long long)s];
      sy += rec[2 * (long long)s + 1];
    }
    out[2 * (long long)i] = sx;
    out[2 * (long long)i + 1] = sy;
  }
}

}  // namespace

void launch_gp2d_wl(const Gp2dWlArgs& a, double* wl_grad, cudaStream_t s) {
  const int nb = grid_blocks(a.n_net, 256, 1024);
  gp2d_wl_kernel<<<nb, 256, 0, s>>>(a);
  gp2d_gather_kernel<<<grid_blocks(a.n_obj, 256, 4096), 256, 0, s>>>(a.n_obj, a.obj_slot_ptr,
                                                                    a.rec, wl_grad);
}

}  // namespace p3d
