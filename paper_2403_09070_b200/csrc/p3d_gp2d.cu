// Multi-die 2D GP (run_gp2d_multi, gp.py:531-690): the
// partial-net weighted-average wirelength over the augmented pin list (each
// HBT joins both partial nets of its crossing net, gp.py:482-498) and its
// per-object owner sums.  Compiled with -fmad=false and written in numpy's
// operation order (wirelength.py:76-98) up to hoisted reciprocals (1/gamma and
// the per-segment 1/s1p, 1/s1m: <= 1 ulp per quotient) and a <= 1.2 ulp
// polynomial exp (numpy's exp is itself <= 1 ulp).
#include <math.h>

#include "p3d_common.cuh"
#include "p3d_internal.cuh"

namespace p3d {

namespace {

// exp(x) for x <= 0 (every WA argument): Cody-Waite reduction by ln 2 and a
// degree-13 Taylor polynomial (<= 1.2 ulp over [-708, 0], the same
// evaluation as K1's exp_neg; numpy's exp is itself <= 1 ulp)
__device__ __forceinline__ double exp_nonpos(double x) {
  const double n = rint(x * 1.4426950408889634074);
  const double r = fma(-n, 1.9082149292705877e-10, fma(-n, 0.693147180369123816490, x));
  double p = 1.6059043836821613e-10;
  p = fma(p, r, 2.08767569878680989792e-09);
  p = fma(p, r, 2.50521083854417187751e-08);
  p = fma(p, r, 2.75573192239858906526e-07);
  p = fma(p, r, 2.75573192239858906526e-06);
  p = fma(p, r, 2.48015873015873015873e-05);
  p = fma(p, r, 1.98412698412698412698e-04);
  p = fma(p, r, 1.38888888888888888889e-03);
  p = fma(p, r, 8.33333333333333333333e-03);
  p = fma(p, r, 4.16666666666666666667e-02);
  p = fma(p, r, 1.66666666666666666667e-01);
  p = fma(p, r, 0.5);
  p = fma(p, r, 1.0);
  p = fma(p, r, 1.0);
  const double sc = __longlong_as_double((long long)((int)n + 1023) << 52);
  return x < -708.0 ? 0.0 : p * sc;
}

struct Seg {
  double hi, lo, s1p, sxp, s1m, sxm, rp, rm, vp, vm;
};

__device__ __forceinline__ double pin_coord(const Gp2dWlArgs& a, int k, int axis) {
  return a.pos[(long long)axis * a.n_obj + a.pin_obj[k]] + (axis ? a.pin_oy[k] : a.pin_ox[k]);
}

// One net, one axis: both (net, die) segments of _segment_wa
// (wirelength.py:76-98) in three passes over the net's pins (extrema, sums in
// pin order, per-pin gradients), 1/gamma and the per-segment reciprocals
// hoisted (<= 1 ulp from numpy's divisions).  Returns the two segments' value.
__device__ __forceinline__ double net_axis(const Gp2dWlArgs& a, int b, int e, int axis,
                                           double ig) {
  Seg sg[2];
#pragma unroll
  for (int d = 0; d < 2; ++d) {
    sg[d].hi = -P3D_INF;
    sg[d].lo = P3D_INF;
    sg[d].s1p = sg[d].sxp = sg[d].s1m = sg[d].sxm = 0.0;
  }
  for (int k = b; k < e; ++k) {
    const double v = pin_coord(a, k, axis);
    Seg& s = sg[a.pin_top[k]];
    s.hi = fmax(s.hi, v);
    s.lo = fmin(s.lo, v);
  }
  for (int k = b; k < e; ++k) {
    const double v = pin_coord(a, k, axis);
    Seg& s = sg[a.pin_top[k]];
    const double ep = exp_nonpos((v - s.hi) * ig), em = exp_nonpos((s.lo - v) * ig);
    s.s1p += ep;
    s.sxp += v * ep;
    s.s1m += em;
    s.sxm += v * em;
  }
  double val = 0.0;
#pragma unroll
  for (int d = 0; d < 2; ++d) {
    Seg& s = sg[d];
    const bool live = s.s1p > 0;
    s.rp = live ? 1.0 / s.s1p : 0.0;
    s.rm = live ? 1.0 / s.s1m : 0.0;
    s.vp = live ? s.sxp * s.rp : 0.0;
    s.vm = live ? s.sxm * s.rm : 0.0;
    val += live ? s.vp - s.vm : 0.0;
  }
  for (int k = b; k < e; ++k) {  // wirelength.py:94-96
    const Seg& s = sg[a.pin_top[k]];
    const double v = pin_coord(a, k, axis);
    const double ep = exp_nonpos((v - s.hi) * ig), em = exp_nonpos((s.lo - v) * ig);
    const double g = ep * s.rp * (1 + (v - s.vp) * ig) - em * s.rm * (1 - (v - s.vm) * ig);
    a.rec[2 * (long long)a.pin_slot[k] + axis] = g;
  }
  return val;
}

__global__ void __launch_bounds__(256) gp2d_wl_kernel(Gp2dWlArgs a) {
  if (a.halt && *a.halt) return;
  __shared__ double red[32];
  double acc[1] = {0.0};
  const double gamma = a.gamma_ptr ? *a.gamma_ptr : a.gamma;
  const double ig = 1.0 / gamma;
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < a.n_net; j += gridDim.x * blockDim.x) {
    const int b = a.net_ptr[j], e = a.net_ptr[j + 1];
    acc[0] += net_axis(a, b, e, 0, ig);
    acc[0] += net_axis(a, b, e, 1, ig);
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
                                                         const double* rec, double* out,
                                                         const int32_t* halt) {
  if (halt && *halt) return;
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
                                                                    a.rec, wl_grad, a.halt);
}

// ---------------------------------------------------------------------------
// the device-resident run_gp2d_multi loop (gp.py:640-681)
// ---------------------------------------------------------------------------
namespace {

enum { kC2Eval = 0, kC2Pre = 1, kC2Adv = 2 };

// gp.py:344-348
__device__ __forceinline__ double clamp_span2(double v, double size, double extent) {
  const double lo = size / 2;
  const double hi = extent - size / 2;
  if (lo <= hi) return clipd(v, lo, hi);
  return dmin(lo, hi) + fabs(hi - lo) / 2;
}

__device__ __forceinline__ void project2(const p3d_gp2d_ctl& c, int i, double& x, double& y) {
  x = clamp_span2(x, c.size_w[i], c.die_w);  // gp.py:571-575
  y = clamp_span2(y, c.size_h[i], c.die_h);
}

__global__ void gp2d_init_kernel(p3d_gp2d_ctl c, const double* pos0) {
  const int O = c.n_obj;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < O; i += gridDim.x * blockDim.x) {
    double x = pos0[i], y = pos0[O + i];
    project2(c, i, x, y);
    c.u[i] = x; c.u[O + i] = y;
    c.v[i] = x; c.v[O + i] = y;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    p3d_gp2d_state* st = c.st;
    st->it = 0;
    st->done = c.max_iters <= 0;
    st->diverged = st->converged = st->lam_set = st->step_set = st->iterations = 0;
    for (int l = 0; l < 3; ++l) {
      st->lam[l] = 0.0;
      st->prev_ovfl[l] = P3D_INF;
    }
    st->step = 0.0;
    st->a = 1.0;
    st->a_new = st->mom = st->dv2_next = st->gmax = 0.0;
    st->gamma = c.max_iters > 0 ? c.gamma_tab[0] : 0.0;
    st->final_overflow = P3D_INF;
    for (int k = 0; k < 8; ++k) st->counters[k] = 0u;
  }
}

// (1) lambda init from the per-layer L1 norms (iteration 0 only,
// gp.py:643-649), the log row and the stop test (gp.py:650-656)
__global__ void __launch_bounds__(256) gp2d_eval_kernel(p3d_gp2d_ctl c) {
  p3d_gp2d_state* st = c.st;
  if (st->done) return;
  __shared__ double red[32 * 6];
  double acc[6] = {0, 0, 0, 0, 0, 0};  // |wl|_1 and |dens|_1 per layer
  const bool need = !st->lam_set;
  if (need) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < c.n_obj; i += gridDim.x * blockDim.x) {
      const int l = c.layer[i];
      const double w = fabs(c.wl_grad[2 * (long long)i]) + fabs(c.wl_grad[2 * (long long)i + 1]);
      const double d = fabs(c.dens_grad[2 * (long long)i]) + fabs(c.dens_grad[2 * (long long)i + 1]);
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        acc[k] += l == k ? w : 0.0;
        acc[3 + k] += l == k ? d : 0.0;
      }
    }
  }
  double* part = c.partials;
  if (need) {
    block_sum<6>(acc, red);
    if (threadIdx.x == 0)
      for (int k = 0; k < 6; ++k) part[k * gridDim.x + blockIdx.x] = acc[k];
  }
  if (!last_block(&st->counters[kC2Eval])) return;
  double tot[6];
  if (need)
    ordered_sums<6>(part, gridDim.x, gridDim.x, red, tot);
  if (threadIdx.x != 0) return;
  if (need) {
    for (int l = 0; l < 3; ++l)  // lambda_init (gp.py:150-153)
      st->lam[l] = (tot[l] <= 0 || tot[3 + l] <= 0) ? 1e-3 : 1e-3 * tot[l] / tot[3 + l];
    st->lam_set = 1;
  }
  const double worst = fmax(fmax(c.ovfl[0], c.ovfl[1]), c.ovfl[2]);
  const int it = st->it;
  st->iterations = it + 1;
  st->final_overflow = worst;
  c.log[4 * it + 0] = it;
  c.log[4 * it + 1] = *c.wl_value;
  c.log[4 * it + 2] = c.n_hbt;
  c.log[4 * it + 3] = worst;
  if (worst <= c.stop_overflow) {  // gp.py:655-656
    st->converged = 1;
    st->done = 1;
  }
}

__device__ __forceinline__ double div2(double lam, double q, double mdeg) {
  double d = lam * q;  // gp.py:142-147 with charges = lam_obj * charges, lam = 1
  d = d + mdeg;
  return dmax(d, 1.0);
}

// (2) the preconditioned gradient of the step and the previous point's raw
// gradient re-weighted by the current lambdas (gp.py:657-667); the BB step
// (or the initial wb / max|g|) and the underflow test (gp.py:198-219)
__global__ void __launch_bounds__(256) gp2d_pre_kernel(p3d_gp2d_ctl c) {
  p3d_gp2d_state* st = c.st;
  if (st->done) return;
  __shared__ double red[32];
  const bool bb = st->step_set != 0;
  const double lam0 = st->lam[0], lam1 = st->lam[1], lam2 = st->lam[2];
  double dg2[1] = {0.0};
  double gm = 0.0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < c.n_obj; i += gridDim.x * blockDim.x) {
    const int l = c.layer[i];
    const double lam = l == 0 ? lam0 : (l == 1 ? lam1 : lam2);
    const double mdeg = c.is_macro[i] ? c.degree[i] : 0.0;
    const double div = div2(lam, c.charge[i], mdeg);
    const long long j = 2 * (long long)i;
    const double wx = c.wl_grad[j], wy = c.wl_grad[j + 1];
    const double dx = c.dens_grad[j], dy = c.dens_grad[j + 1];
    const double px = (wx + lam * dx) / div, py = (wy + lam * dy) / div;
    if (bb) {
      const double qx = (c.prev_wl[j] + lam * c.prev_dens[j]) / div;
      const double qy = (c.prev_wl[j + 1] + lam * c.prev_dens[j + 1]) / div;
      const double ex = px - qx, ey = py - qy;
      dg2[0] += ex * ex + ey * ey;
    } else {
      gm = fmax(gm, fmax(fabs(px), fabs(py)));
    }
    c.pre[j] = px;
    c.pre[j + 1] = py;
    c.prev_wl[j] = wx;
    c.prev_wl[j + 1] = wy;
    c.prev_dens[j] = dx;
    c.prev_dens[j + 1] = dy;
  }
  double* part = c.partials;
  if (bb) {
    block_sum<1>(dg2, red);
    if (threadIdx.x == 0) part[blockIdx.x] = dg2[0];
  } else {
    gm = block_max(gm, red);
    if (threadIdx.x == 0) part[blockIdx.x] = gm;
  }
  if (!last_block(&st->counters[kC2Pre])) return;
  double v;
  if (bb) v = ordered_sum(part, gridDim.x, red);
  else v = block_max_partials((volatile double*)part, gridDim.x, red);
  if (threadIdx.x != 0) return;
  if (!bb) {  // NesterovOptimizer._init_step (gp.py:198-202)
    st->gmax = v;
    st->step = v == 0.0 ? 1.0 : c.step_scale / v;
    st->step_set = 1;
  } else {
    const double den = sqrt(v);  // gp.py:210-217
    if (den > 0) {
      const double nw = sqrt(st->dv2_next) / den;
      st->step = fmin(fmax(nw, st->step / 4), st->step * 4);
    }
  }
  if (!isfinite(st->step) || st->step <= c.min_step) {  // StepUnderflow (gp.py:218-219, 672)
    st->diverged = 1;
    st->done = 1;
    return;
  }
  const double a = st->a;
  st->a_new = (1 + sqrt(4 * (a * a) + 1)) / 2;
  st->mom = (a - 1) / st->a_new;
}

// (3) u' = P(v - s g), v' = P(u' + m (u' - u)) (gp.py:220-227); last block:
// per-layer mu / lambda update (gp.py:678-681) and the next gamma
__global__ void __launch_bounds__(256) gp2d_adv_kernel(p3d_gp2d_ctl c) {
  p3d_gp2d_state* st = c.st;
  if (st->done) return;
  __shared__ double red[32];
  const int O = c.n_obj;
  const double step = st->step, mom = st->mom;
  double dv2[1] = {0.0};
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < O; i += gridDim.x * blockDim.x) {
    const double ux = c.u[i], uy = c.u[O + i], vx = c.v[i], vy = c.v[O + i];
    double nx = vx - step * c.pre[2 * (long long)i], ny = vy - step * c.pre[2 * (long long)i + 1];
    project2(c, i, nx, ny);
    double mx = nx + mom * (nx - ux), my = ny + mom * (ny - uy);
    project2(c, i, mx, my);
    const double ex = mx - vx, ey = my - vy;
    dv2[0] += ex * ex + ey * ey;
    c.u[i] = nx; c.u[O + i] = ny;
    c.v[i] = mx; c.v[O + i] = my;
  }
  block_sum<1>(dv2, red);
  if (threadIdx.x == 0) c.partials[blockIdx.x] = dv2[0];
  if (!last_block(&st->counters[kC2Adv])) return;
  const double tot = ordered_sum(c.partials, gridDim.x, red);
  if (threadIdx.x != 0) return;
  st->dv2_next = tot;
  st->a = st->a_new;
  for (int l = 0; l < 3; ++l) {  // mu_from_overflow (gp.py:156-168)
    const double drop = st->prev_ovfl[l] - c.ovfl[l];
    double mu;
    if (drop < 0) mu = c.mu_min;
    else if (drop >= 2e-3) mu = c.mu_min + 0.01;
    else if (drop >= 5e-4) mu = (c.mu_min + c.mu_max) / 2;
    else mu = c.mu_max;
    mu = fmin(fmax(mu, c.mu_min), c.mu_max);
    st->lam[l] *= mu;
    st->prev_ovfl[l] = c.ovfl[l];
  }
  st->it += 1;
  if (st->it >= c.max_iters) st->done = 1;
  else st->gamma = c.gamma_tab[st->it];
}

__global__ void gp2d_project_kernel(p3d_gp2d_ctl c, const double* in, double* out) {
  const int O = c.n_obj;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < O; i += gridDim.x * blockDim.x) {
    double x = in[i], y = in[O + i];
    project2(c, i, x, y);
    out[i] = x;
    out[O + i] = y;
  }
}

__global__ void gp2d_layer_xy_kernel(int n, const int32_t* idx, const double* pos, int n_obj,
                                     double* x, double* y, const int32_t* halt) {
  if (halt && *halt) return;
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
    const int i = idx[k];
    x[k] = pos[i];
    y[k] = pos[n_obj + i];
  }
}

__global__ void gp2d_layer_force_kernel(int n, const int32_t* idx, const double* force,
                                        double* dens_grad, const int32_t* halt) {
  if (halt && *halt) return;
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
    const long long i = idx[k];
    dens_grad[2 * i] = force[3 * (long long)k];
    dens_grad[2 * i + 1] = force[3 * (long long)k + 1];
  }
}

}  // namespace

int gp2d_init(const p3d_gp2d_ctl& c, const double* pos0, cudaStream_t s) {
  gp2d_init_kernel<<<grid_blocks(c.n_obj, 256, 1024), 256, 0, s>>>(c, pos0);
  return check_launch("gp2d_init");
}

int gp2d_step(const p3d_gp2d_ctl& c, cudaStream_t s) {
  gp2d_eval_kernel<<<c.nblk, 256, 0, s>>>(c);
  gp2d_pre_kernel<<<c.nblk, 256, 0, s>>>(c);
  gp2d_adv_kernel<<<c.nblk, 256, 0, s>>>(c);
  return check_launch("gp2d_step");
}

int gp2d_project(const p3d_gp2d_ctl& c, const double* in, double* out, cudaStream_t s) {
  gp2d_project_kernel<<<grid_blocks(c.n_obj, 256, 1024), 256, 0, s>>>(c, in, out);
  return check_launch("gp2d_project");
}

void launch_gp2d_layer_xy(int n, const int32_t* idx, const double* pos, int n_obj, double* x,
                          double* y, const int32_t* halt, cudaStream_t s) {
  gp2d_layer_xy_kernel<<<grid_blocks(n, 256, 1024), 256, 0, s>>>(n, idx, pos, n_obj, x, y, halt);
}

void launch_gp2d_layer_force(int n, const int32_t* idx, const double* force, double* dens_grad,
                             const int32_t* halt, cudaStream_t s) {
  gp2d_layer_force_kernel<<<grid_blocks(n, 256, 1024), 256, 0, s>>>(n, idx, force, dens_grad, halt);
}

}  // namespace p3d
