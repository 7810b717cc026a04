// The device-resident GP iteration (gp.py:359-455 run_gp3d), K4 (fused with
// the objective assembly) and K5 (preconditioner + Nesterov/BB step).
// Compiled with -fmad=false so the optimiser arithmetic rounds exactly like
// numpy's (no contracted v - step*g etc.).
//
// Kernel sequence of one iteration (each a no-op once st->done is set):
//   K1  net_kernel      WL value/grads per pin (slot order), exact WL, crossings
//   K1b gather_kernel   per-instance sums, L1 norms, Eq. 17 scale
//   K2  scatter         fixed-point rho (cells thread-per-object, macro per CTA)
//   K3  spectral        phi/E maps; the first pass also yields the overflow
//                       and re-zeroes rho for the next iteration
//   K4  dens_kernel     density means -> dens grad; WL grad assembly; energy;
//                       preconditioned current and re-weighted previous
//                       gradient (Eq. 19) and the BB norms |dv|, |dg|;
//                       last block: objective, lambda init, log row, best key,
//                       stop / divergence tests, BB step, underflow test
//                       (gp.py:386-437)
//   K5a gmax0_kernel    iteration 0 only: max|g| for the initial step
//                       (gp.py:198-202, needs the just-initialised lambda)
//   K5b advance_kernel  best snapshot; u' = P(v - s g), v' = P(u' + m (u' - u))
//                       with g re-derived from the stored gradients; last
//                       block: mu schedule, lambda update, next gamma
//                       (gp.py:220-227, 442-444)
#include <math.h>
#include <stdlib.h>

#include "p3d_geom.cuh"
#include "p3d_internal.cuh"

namespace p3d {

template <class Cloud>
void launch_scatter(const Cloud& cl, int n, int n_macro, const int32_t* macro_ids,
                    const p3d_grid& g, int64_t* rho, const int* halt, cudaStream_t s);

__device__ __forceinline__ double* fin(const p3d_gp& gp) {
  return gp.partials + (long long)kSlotFinal * kPartialStride;
}

// this rank's objects (all of them on one GPU): local index k -> object index
__host__ __device__ __forceinline__ int own_count(const p3d_gp& gp) {
  return (gp.sh_i1 - gp.sh_i0) + (gp.sh_f1 - gp.sh_f0);
}
__device__ __forceinline__ int own_obj(const p3d_gp& gp, int k) {
  const int ni = gp.sh_i1 - gp.sh_i0;
  return k < ni ? gp.sh_i0 + k : gp.sh_f0 + (k - ni);
}

__device__ __forceinline__ CloudGP cloud_of(const p3d_gp& gp, const double* pos) {
  CloudGP c;
  c.pos = pos;
  c.n_inst = gp.n_inst;
  c.n_obj = gp.n_obj;
  c.wt = gp.w_top; c.ht = gp.h_top; c.wb = gp.w_bot; c.hb = gp.h_bot;
  c.fw = gp.fill_w; c.fh = gp.fill_h;
  c.macro = gp.is_macro;
  c.dz = gp.grid.dz;
  c.target_density = gp.target_density;
  return c;
}

// gp.py:344-348
__device__ __forceinline__ double clamp_span(double v, double size, double extent) {
  const double lo = size / 2;
  const double hi = extent - size / 2;
  if (lo <= hi) return clipd(v, lo, hi);
  return dmin(lo, hi) + fabs(hi - lo) / 2;
}

// Gp3dProblem.project for one object (gp.py:280-294)
__device__ __forceinline__ void project_obj(const p3d_gp& gp, int i, double& x, double& y,
                                            double& z) {
  const double dz = gp.grid.dz;
  if (i < gp.n_inst) {
    z = clipd(z, dz / 4, 3 * dz / 4);
    double w, h;
    dynamic_wh(z, dz, gp.is_macro[i] != 0, gp.w_top[i], gp.h_top[i], gp.w_bot[i], gp.h_bot[i],
               w, h);
    x = clamp_span(x, w, gp.grid.dx);
    y = clamp_span(y, h, gp.grid.dy);
  } else {
    const int f = i - gp.n_inst;
    x = clamp_span(x, gp.fill_w[f], gp.grid.dx);
    y = clamp_span(y, gp.fill_h[f], gp.grid.dy);
    z = gp.fill_z[f];
  }
}

__global__ void project_kernel(p3d_gp gp, const double* in, double* out) {
  const int O = gp.n_obj;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < O; i += gridDim.x * blockDim.x) {
    double x = in[i], y = in[O + i], z = in[2 * O + i];
    project_obj(gp, i, x, y, z);
    out[i] = x;
    out[O + i] = y;
    out[2 * O + i] = z;
  }
}

// ---------------------------------------------------------------------------
// loop state init / eval setup
// ---------------------------------------------------------------------------
__global__ void init_state_kernel(p3d_gp gp) {
  p3d_loop_state* st = gp.st;
  st->it = 0;
  st->done = gp.max_iters <= 0;
  st->diverged = 0;
  st->lam_set = 0;
  st->step_set = 0;
  st->stop_now = 0;
  st->best_flag = 0;
  st->rise = 0;
  st->nonfinite = 0;
  st->converged = 0;
  st->eval_only = 0;
  st->lam = 0.0;
  st->a = 1.0;
  st->step = 0.0;
  st->prev_ovfl = P3D_INF;
  st->prev_value = P3D_INF;
  st->dv2_next = 0.0;
  st->last_mu = 1.0;
  st->best0 = P3D_INF;
  st->best1 = P3D_INF;
  st->gamma = gp.max_iters > 0 ? gp.gamma_tab[0] : 0.0;
  st->lam_eval = 0.0;
  st->iterations = 0;
  st->hbt_count = 0;
  st->final_overflow = P3D_INF;
  st->wirelength = 0.0;
  for (int k = 0; k < 16; ++k) st->counters[k] = 0u;
}

__global__ void eval_setup_kernel(p3d_gp gp, double lam, double gamma) {
  p3d_loop_state* st = gp.st;
  st->eval_only = 1;
  st->done = 0;
  st->lam_eval = lam;
  st->gamma = gamma;
}

__global__ void copy3_kernel(int O, const double* a, double* b, double* c) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < 3 * O; i += gridDim.x * blockDim.x) {
    const double v = a[i];
    b[i] = v;
    if (c) c[i] = v;
  }
}

// AoS copy of the instance centres for the K1 pin gathers
__global__ void pos4_kernel(int I, int O, const double* v, double* pos4) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < I; i += gridDim.x * blockDim.x)
    reinterpret_cast<double4*>(pos4)[i] = make_double4(v[i], v[O + i], v[2 * O + i], 0.0);
}

// ---------------------------------------------------------------------------
// K4: density gather + objective assembly; last block = loop control part 1
// ---------------------------------------------------------------------------
__device__ __forceinline__ double precond_div(double lam, double q, double mdeg) {
  double d = lam * q;  // gp.py:142-147 operation order
  d = d + mdeg;
  return dmax(d, 1.0);
}

#ifndef P3D_K4_KEEP
#define P3D_K4_KEEP 1
#endif
// P3D_PRE_STORE: K4 stores the preconditioned gradient the step uses (K5 reads
// 24 B per object instead of re-deriving it from 56 B of raw gradients) and
// this point's gradient re-weighted under the NEXT lambda, which is known here
// already: lambda_{t+1} = lambda_t mu(ovfl_{t-1}, ovfl_t), and ovfl_t comes
// from K3.  So K4 reads 24 B of re-weighted previous gradient instead of 56 B
// of raw ones.  Same operations on the same operands: bit-identical iterates.
// Iteration 0 (lambda set by K4's own reduction) keeps the raw gradients and
// gmax0_kernel converts them in place.
#ifndef P3D_PRE_STORE
#define P3D_PRE_STORE 1
#endif

// mu_from_overflow (gp.py:156-168)
__device__ __forceinline__ double mu_of(const p3d_gp& gp, double prev_ovfl, double ovfl) {
  const double drop = prev_ovfl - ovfl;
  double mu;
  if (drop < 0) mu = gp.mu_min;
  else if (drop >= 2e-3) mu = gp.mu_min + 0.01;
  else if (drop >= 5e-4) mu = (gp.mu_min + gp.mu_max) / 2;
  else mu = gp.mu_max;
  return fmin(fmax(mu, gp.mu_min), gp.mu_max);
}
#ifndef P3D_K4_LDCS
#define P3D_K4_LDCS 0
#endif
// per-launch scalars of K4 (the loop state changes only in the last block,
// after every object has been processed)
struct DensScal {
  double lam, zscale, lam_next;
  bool eval_only, bb;
};

// acc: energy, |dens|_1, |wl|_1, non-finite count, (unused), |dg|^2
// wl4 = the object's owner sums (gx, gy, g_cut, FD), pw/pd/pq its previous raw
// gradients and charge: loaded by the caller before the map gathers so their
// latency overlaps them.
__device__ __forceinline__ void finish_object(const p3d_gp& gp, int i, const Charge& q,
                                              const double (&mean)[4], const DensScal& sc,
                                              const double (&wl4)[4], const double (&pw)[3],
                                              const double (&pd)[3], double pq, double mdeg,
                                              double (&acc)[6]) {
  const int O = gp.n_obj, I = gp.n_inst;
  const double qq = charge_of(q);
  const double c = -2.0 * qq;
  double dg[3] = {mean[1] * c, mean[2] * c, i < I ? mean[3] * c : 0.0};  // filler z frozen
  double wl[3] = {0.0, 0.0, 0.0};
  if (i < I) {
    wl[0] = wl4[0];
    wl[1] = wl4[1];
    wl[2] = sc.zscale * wl4[3] + gp.alpha * wl4[2];  // wirelength.py:296-305
  }
  const double lam = sc.lam;
  bool finite = true;
#pragma unroll
  for (int k = 0; k < 3; ++k) finite = finite && isfinite(wl[k] + lam * dg[k]);
  acc[0] += qq * mean[0];
  acc[1] += fabs(dg[0]) + fabs(dg[1]) + fabs(dg[2]);
  acc[2] += fabs(wl[0]) + fabs(wl[1]) + fabs(wl[2]);
  acc[3] += finite ? 0.0 : 1.0;
  if (sc.eval_only) {
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      gp.wl_grad[(long long)k * O + i] = wl[k];
      gp.dens_grad[(long long)k * O + i] = dg[k];
    }
    return;
  }
  // BB denominator: the previous iteration's raw gradients re-weighted by the
  // current lambda (gp.py:427-435); at iteration 0 there is no previous point.
  // (The numerator |v - v_prev|^2 comes from the last advance.)
#if P3D_PRE_STORE
  if (sc.bb) {  // pw = this point's predecessor, re-weighted under lam (last K4)
    const double div = precond_div(lam, qq, mdeg);
    const double ydiv = 1.0 / div;
    const double lamn = sc.lam_next;
    const double divn = precond_div(lamn, qq, mdeg);
    const double ydivn = 1.0 / divn;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      const double pre = div_rcp(wl[k] + lam * dg[k], div, ydiv);
      const double d = pre - pw[k];
      acc[5] += d * d;
      const double ppn = div_rcp(wl[k] + lamn * dg[k], divn, ydivn);
#if P3D_K4_KEEP
      st_keep(gp.prev_wl + (long long)k * O + i, pre);
      st_keep(gp.prev_dens + (long long)k * O + i, ppn);
#else
      gp.prev_wl[(long long)k * O + i] = pre;
      gp.prev_dens[(long long)k * O + i] = ppn;
#endif
    }
    return;
  }
#else
  if (sc.bb) {
    const double div = precond_div(lam, qq, mdeg);
    const double divp = precond_div(lam, pq, mdeg);
    const double ydiv = 1.0 / div, ydivp = 1.0 / divp;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      const double pre = div_rcp(wl[k] + lam * dg[k], div, ydiv);
      const double pp = div_rcp(pw[k] + lam * pd[k], divp, ydivp);
      const double d = pre - pp;
      acc[5] += d * d;
    }
  }
#endif
#if P3D_K4_KEEP  // K5 reads these right after: keep them in L2
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    st_keep(gp.prev_wl + (long long)k * O + i, wl[k]);
    st_keep(gp.prev_dens + (long long)k * O + i, dg[k]);
  }
  st_keep(gp.prev_q + i, qq);
#else
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    gp.prev_wl[(long long)k * O + i] = wl[k];
    gp.prev_dens[(long long)k * O + i] = dg[k];
  }
  gp.prev_q[i] = qq;
#endif
}

// the caller-side loads of finish_object's inputs
__device__ __forceinline__ void load_object_inputs(const p3d_gp& gp, int i, const DensScal& sc,
                                                   double (&wl4)[4], double (&pw)[3],
                                                   double (&pd)[3], double& pq, double& mdeg) {
  const int O = gp.n_obj, I = gp.n_inst;
  wl4[0] = wl4[1] = wl4[2] = wl4[3] = 0.0;
  if (i < I) {
#pragma unroll
    {
#if P3D_K4_LDCS  // read once: evict first
      const double2* g2 = reinterpret_cast<const double2*>(gp.inst_g) + 2 * (long long)i;
      const double2 ga = __ldcs(g2), gb = __ldcs(g2 + 1);
      wl4[0] = ga.x; wl4[1] = ga.y; wl4[2] = gb.x; wl4[3] = gb.y;
#else
      const double4 g = reinterpret_cast<const double4*>(gp.inst_g)[i];
      wl4[0] = g.x; wl4[1] = g.y; wl4[2] = g.z; wl4[3] = g.w;
#endif
    }
  }
  pq = mdeg = 0.0;
  pw[0] = pw[1] = pw[2] = pd[0] = pd[1] = pd[2] = 0.0;
  if (sc.bb && !sc.eval_only) {
#if P3D_PRE_STORE
#pragma unroll
    for (int k = 0; k < 3; ++k) pw[k] = gp.prev_dens[(long long)k * O + i];
#else
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      pw[k] = gp.prev_wl[(long long)k * O + i];
      pd[k] = gp.prev_dens[(long long)k * O + i];
    }
    pq = gp.prev_q[i];
#endif
    mdeg = (i < I && gp.is_macro[i]) ? gp.degree[i] : 0.0;
  }
}

// underflow test and momentum of the accepted step (gp.py:218-226)
__device__ __forceinline__ void step_tail(const p3d_gp& gp) {
  p3d_loop_state* st = gp.st;
  if (!isfinite(st->step) || st->step <= gp.min_step) {  // StepUnderflow, gp.py:438-441
    st->diverged = 1;
    st->stop_now = 1;  // the best snapshot of this iteration is still taken
    return;
  }
  const double a = st->a;
  st->a_new = (1 + sqrt(4 * (a * a) + 1)) / 2;
  st->mom = (a - 1) / st->a_new;
}

__device__ __forceinline__ void control_after_eval(const p3d_gp& gp, double energy, double l1_dens,
                                   double l1_wl, double nonfinite, double dv2, double dg2) {
  p3d_loop_state* st = gp.st;
  // one thread on the critical path of every iteration: every state scalar it
  // reads is loaded up front, so the control below costs one round trip
  // rather than a chain of dependent ones
  const double* f = fin(gp);
  const double f0 = f[kFinNet + 0], f1 = f[kFinNet + 1], f2 = f[kFinNet + 2];
  const double f3 = f[kFinNet + 3], f4 = f[kFinNet + 4], f5 = f[kFinNet + 5];
  const double fov = f[kFinOvfl];
  const double n0 = f[kFinNorm + 0], n1 = f[kFinNorm + 1], n2 = f[kFinNorm + 2];
  const double n3 = f[kFinNorm + 3];
  const double lam_eval = st->lam_eval;
  const bool eval_only = st->eval_only != 0, lam_set = st->lam_set != 0;
  const bool step_set = st->step_set != 0;
  const int it = st->it, rise0 = st->rise;
  const double best0 = st->best0, best1 = st->best1, prev_value = st->prev_value;
  const double last_mu = st->last_mu, dv2_next = st->dv2_next, step0 = st->step, a0 = st->a;
  const int W = gp.divergence_window;
  const int first = W > 0 ? it - W + 1 : 0;
  const double hist_first = (first >= 0 && first < it) ? gp.ovfl_hist[first] : 0.0;
  const double wl_bi = f0 + f1;
  const double cut = f2;
  const double exact = f3 + f4;
  const double ncross = f5;
  const double ovfl = gp.movable_volume <= 0 ? 0.0 : fov;
  const double wl_value = wl_bi + gp.alpha * cut;
  double value = wl_bi + gp.alpha * cut + lam_eval * energy;  // gp.py:326
  st->wl_x = f0;
  st->wl_y = f1;
  st->cut = cut;
  st->exact = exact;
  st->ncross = ncross;
  st->norm_x = n0;
  st->norm_y = n1;
  st->norm_zb = n2;
  st->gz_scale = n3;
  st->energy = energy;
  st->ovfl = ovfl;
  st->wl_value = wl_value;
  st->l1_wl = l1_wl;
  st->l1_dens = l1_dens;
  st->nonfinite = nonfinite != 0.0;
  st->value = value;
  if (eval_only) {
    st->done = 1;
    return;
  }
  if (!isfinite(value) || nonfinite != 0.0) {  // gp.py:328-329, 390-393
    st->diverged = 1;
    st->done = 1;
    return;
  }
  if (!lam_set) {  // gp.py:394-399, lambda_init gp.py:150-153
    const double lam = (l1_wl <= 0 || l1_dens <= 0) ? 1e-3 : 1e-3 * l1_wl / l1_dens;
    st->lam = lam;
    st->lam_set = 1;
    value = wl_value + lam * energy;
    st->value = value;
  }
  gp.log[4 * it + 0] = it;
  gp.log[4 * it + 1] = exact;
  gp.log[4 * it + 2] = ncross;
  gp.log[4 * it + 3] = ovfl;
  st->iterations = it + 1;
  st->final_overflow = ovfl;
  st->wirelength = exact;
  st->hbt_count = (int)ncross;
  const double k0 = fmax(ovfl - gp.stop_overflow, 0.0);  // gp.py:406-409
  if (k0 < best0 || (k0 == best0 && value < best1)) {
    st->best0 = k0;
    st->best1 = value;
    st->best_flag = 1;
  }
  if (ovfl <= gp.stop_overflow) {  // gp.py:410-411
    st->converged = 1;
    st->stop_now = 1;
    return;
  }
  const int rise = value > prev_value * last_mu ? rise0 + 1 : 0;  // gp.py:414-422
  st->rise = rise;
  st->prev_value = value;
  gp.ovfl_hist[it] = ovfl;
  if (rise >= W) {
    const double hf = first == it ? ovfl : hist_first;
    if (hf - ovfl < 1e-3) {
      st->diverged = 1;
      st->stop_now = 1;
      return;
    }
  }
  st->dv2 = dv2_next;  // |v - v_prev|^2, accumulated by the last advance
  st->dg2 = dg2;
  dv2 = dv2_next;
  if (!step_set) return;  // iteration 0: gmax0_kernel sets the initial step
  double step = step0;
  const double den = sqrt(dg2);  // gp.py:210-217
  if (den > 0) {
    const double bb = sqrt(dv2) / den;
    step = fmin(fmax(bb, step0 / 4), step0 * 4);
    st->step = step;
  }
  // step_tail (gp.py:218-226, 438-441) on the values in registers
  if (!isfinite(step) || step <= gp.min_step) {
    st->diverged = 1;
    st->stop_now = 1;  // the best snapshot of this iteration is still taken
    return;
  }
  const double a_new = (1 + sqrt(4 * (a0 * a0) + 1)) / 2;
  st->a_new = a_new;
  st->mom = (a0 - 1) / a_new;
}

#ifndef P3D_K4_PREFETCH
#define P3D_K4_PREFETCH 0
#endif
#ifndef P3D_K4_MINB
#define P3D_K4_MINB 4
#endif
__global__ void __launch_bounds__(256, P3D_K4_MINB) dens_kernel(p3d_gp gp) {
  pdl_wait();
  const p3d_loop_state* st = gp.st;
  if (st->done) return;
  __shared__ double red[32 * 6];
  DensScal sc;
  sc.lam = st->lam_eval;
  sc.eval_only = st->eval_only != 0;
  sc.bb = st->step_set != 0;
  {
    const double* f = fin(gp);
    sc.zscale = f[kFinNorm + 2] == 0.0 ? 0.0 : f[kFinNorm + 3];  // Eq. 17 (0 if |gz| = 0)
    // lambda of the next iteration, exactly as advance_kernel will form it
    const double ovfl = gp.movable_volume <= 0 ? 0.0 : f[kFinOvfl];
    sc.lam_next = sc.lam * mu_of(gp, st->prev_ovfl, ovfl);
  }
  const CloudGP cl = cloud_of(gp, gp.v);
  double acc[6] = {0, 0, 0, 0, 0, 0};
  const int nm = gp.n_macro;
  if ((int)blockIdx.x < nm) {
    const int i = gp.macro_ids[blockIdx.x];
    const Charge q = cl.get(i);
    double mean[4];
    gather_object_block(q, gp.grid, gp.maps, mean, red);
    if (threadIdx.x == 0) {
      double wl4[4], pw[3], pd[3], pq, mdeg;
      load_object_inputs(gp, i, sc, wl4, pw, pd, pq, mdeg);
      finish_object(gp, i, q, mean, sc, wl4, pw, pd, pq, mdeg, acc);
    }
  } else {
    const int b = blockIdx.x - nm, nb = gridDim.x - nm, n_own = own_count(gp);
    for (int k = b * blockDim.x + threadIdx.x; k < n_own; k += nb * blockDim.x) {
      const int i = own_obj(gp, k);
      const Charge q = cl.get(i);  // reads the macro flag too: one round trip
      if (cl.is_macro(i)) continue;
      double wl4[4], pw[3], pd[3], pq, mdeg;
#if P3D_K4_PREFETCH
      load_object_inputs(gp, i, sc, wl4, pw, pd, pq, mdeg);
#endif
      double mean[4];
      gather_object(q, gp.grid, gp.maps, mean);
#if !P3D_K4_PREFETCH
      load_object_inputs(gp, i, sc, wl4, pw, pd, pq, mdeg);
#endif
      finish_object(gp, i, q, mean, sc, wl4, pw, pd, pq, mdeg, acc);
    }
  }
  double* part = gp.partials + (long long)kSlotDens * kPartialStride;
  block_sum<6>(acc, red);
  if (threadIdx.x == 0)
    for (int k = 0; k < 6; ++k) part[k * gridDim.x + blockIdx.x] = acc[k];
  if (last_block(&gp.st->counters[kCntDens])) {
    double tot[6];
    ordered_sums<6>(part, gridDim.x, gridDim.x, red, tot);
    if (threadIdx.x == 0) {
      if (gp.shard_size > 0) {  // sharded: the host all-reduces, then shard_control_kernel
        for (int k = 0; k < 6; ++k) gp.shard_tot[8 + k] = tot[k];
      } else {
        control_after_eval(gp, tot[0], tot[1], tot[2], tot[3], tot[4], tot[5]);
      }
    }
  }
}

// ---------------------------------------------------------------------------
// K5a: iteration 0 only — max |g| of the preconditioned gradient under the
// just-initialised lambda, then the initial step wb / max|g| (gp.py:198-202)
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) gmax0_kernel(p3d_gp gp) {
  pdl_wait();
  p3d_loop_state* st = gp.st;
  if (st->done || st->step_set || st->stop_now) return;
  __shared__ double red[32];
  const int O = gp.n_obj, I = gp.n_inst;
  const double lam = st->lam;
#if P3D_PRE_STORE
  const double lam1 = lam * mu_of(gp, st->prev_ovfl, st->ovfl);  // as advance_kernel forms it
#endif
  double m = 0.0;
  const int n_own = own_count(gp);
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n_own; k += gridDim.x * blockDim.x) {
    const int i = own_obj(gp, k);
    const double mdeg = (i < I && gp.is_macro[i]) ? gp.degree[i] : 0.0;
    const double div = precond_div(lam, gp.prev_q[i], mdeg);
#if P3D_PRE_STORE  // the raw gradients of iteration 0 -> (pre, re-weighted under lambda_1)
    const double ydiv = 1.0 / div;
    const double divn = precond_div(lam1, gp.prev_q[i], mdeg), ydivn = 1.0 / divn;
#endif
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      const long long j = (long long)k * O + i;
      m = fmax(m, fabs((gp.prev_wl[j] + lam * gp.prev_dens[j]) / div));
#if P3D_PRE_STORE
      const double w = gp.prev_wl[j], d = gp.prev_dens[j];
      gp.prev_wl[j] = div_rcp(w + lam * d, div, ydiv);
      gp.prev_dens[j] = div_rcp(w + lam1 * d, divn, ydivn);
#endif
    }
  }
  double* part = gp.partials + (long long)kSlotStep * kPartialStride;
  m = block_max(m, red);
  if (threadIdx.x == 0) part[blockIdx.x] = m;
  if (last_block(&st->counters[kCntStep])) {
    const double gm = block_max_partials((volatile double*)part, gridDim.x, red);
    if (threadIdx.x == 0) {
      if (gp.shard_size > 0) {  // sharded: max over ranks, then step0_control_kernel
        gp.shard_tot[16] = gm;
      } else {
        st->gmax = gm;
        st->step = gm == 0.0 ? 1.0 : gp.step_scale / gm;
        st->step_set = 1;
        step_tail(gp);
      }
    }
  }
}

// ---------------------------------------------------------------------------
// K5b: projected Nesterov update (gp.py:220-227); last block: schedules
// ---------------------------------------------------------------------------
#ifndef P3D_K5_MINB
#define P3D_K5_MINB 3
#endif
// project_obj (gp.py:280-294) on sizes loaded up front (same arithmetic)
__device__ __forceinline__ void project_loaded(const p3d_gp& gp, bool inst, bool mac, double s0,
                                               double s1, double s2, double s3, double fz,
                                               double& x, double& y, double& z) {
  const double dz = gp.grid.dz;
  if (inst) {
    z = clipd(z, dz / 4, 3 * dz / 4);
    double w, h;
    dynamic_wh(z, dz, mac, s0, s1, s2, s3, w, h);
    x = clamp_span(x, w, gp.grid.dx);
    y = clamp_span(y, h, gp.grid.dy);
  } else {
    x = clamp_span(x, s0, gp.grid.dx);
    y = clamp_span(y, s1, gp.grid.dy);
    z = fz;
  }
}

// Every input of an object is loaded before the first store (read-only data
// through the non-coherent path), so one object costs one memory round trip.
__global__ void __launch_bounds__(256, P3D_K5_MINB) advance_kernel(p3d_gp gp) {
  pdl_wait();
  p3d_loop_state* st = gp.st;
  if (st->done) return;
  __shared__ double red[32];
  const int O = gp.n_obj, I = gp.n_inst;
  const bool best = st->best_flag != 0, stop = st->stop_now != 0;
  const double step = st->step, mom = st->mom, lam = st->lam;
  if (!stop && !st->step_set) {  // no initial step: p3d_gp_iterate_steady at iteration 0
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      st->diverged = 1;
      st->done = 1;
    }
    return;
  }
  double dv2[1] = {0.0};
  const int n_own = own_count(gp);
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n_own; k += gridDim.x * blockDim.x) {
    const int i = own_obj(gp, k);
    const bool inst = i < I;
    double u[3], v[3], pw[3];
#if !P3D_PRE_STORE
    double pd[3];
#endif
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const long long j = (long long)c * O + i;
      u[c] = gp.u[j];
      v[c] = gp.v[j];
      pw[c] = __ldg(gp.prev_wl + j);  // P3D_PRE_STORE: the preconditioned gradient
#if !P3D_PRE_STORE
      pd[c] = __ldg(gp.prev_dens + j);
#endif
    }
#if !P3D_PRE_STORE
    const double pq = __ldg(gp.prev_q + i);
#endif
    bool mac = false;
    double s0, s1, s2 = 0.0, s3 = 0.0, fz = 0.0, mdeg = 0.0;
    if (inst) {
      mac = __ldg(gp.is_macro + i) != 0;
      s0 = __ldg(gp.w_top + i);
      s1 = __ldg(gp.h_top + i);
      s2 = __ldg(gp.w_bot + i);
      s3 = __ldg(gp.h_bot + i);
#if !P3D_PRE_STORE
      if (mac) mdeg = __ldg(gp.degree + i);
#endif
    } else {
      const int f = i - I;
      s0 = __ldg(gp.fill_w + f);
      s1 = __ldg(gp.fill_h + f);
      fz = __ldg(gp.fill_z + f);
    }
    if (best) {  // gp.py:406-409 (taken before the stop / advance, as in the reference)
#pragma unroll
      for (int c = 0; c < 3; ++c) gp.best[(long long)c * O + i] = u[c];
    }
    if (stop) continue;
    double un[3], vn[3];
#if P3D_PRE_STORE
    (void)mdeg;
    (void)lam;
#pragma unroll
    for (int c = 0; c < 3; ++c) un[c] = v[c] - step * pw[c];
#else
    // the step's gradient, re-derived from the stored raw gradients (gp.py:424-426)
    const double div = precond_div(lam, pq, mdeg);
    const double ydiv = 1.0 / div;
#pragma unroll
    for (int c = 0; c < 3; ++c) un[c] = v[c] - step * div_rcp(pw[c] + lam * pd[c], div, ydiv);
#endif
    project_loaded(gp, inst, mac, s0, s1, s2, s3, fz, un[0], un[1], un[2]);
#pragma unroll
    for (int c = 0; c < 3; ++c) vn[c] = un[c] + mom * (un[c] - u[c]);
    project_loaded(gp, inst, mac, s0, s1, s2, s3, fz, vn[0], vn[1], vn[2]);
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const long long j = (long long)c * O + i;
      const double d = vn[c] - v[c];  // BB numerator of the next evaluation (gp.py:210)
      dv2[0] += d * d;
      gp.u[j] = un[c];
      gp.v[j] = vn[c];
    }
    if (inst) {  // K1 gathers these next iteration: keep them in L2
      st_keep2(gp.pos4 + 4 * (long long)i, vn[0], vn[1]);
      st_keep2(gp.pos4 + 4 * (long long)i + 2, vn[2], 0.0);
    }
  }
  double* part = gp.partials + (long long)kSlotAdv * kPartialStride;
  block_sum<1>(dv2, red);
  if (threadIdx.x == 0) part[blockIdx.x] = dv2[0];
  if (last_block(&st->counters[kCntAdvance])) {
    const double tot = ordered_sum(part, gridDim.x, red);
    if (threadIdx.x == 0) {
      if (stop) {
        st->done = 1;
        return;
      }
      st->dv2_next = tot;
      // sharded: this rank's share; it rides along the next iteration's
      // density-totals all-reduce (shard_control_kernel reads the sum)
      if (gp.shard_size > 0) gp.shard_tot[14] = tot;
      st->a = st->a_new;
      // mu_from_overflow (gp.py:156-168), lambda update (gp.py:442-444)
      const double mu = mu_of(gp, st->prev_ovfl, st->ovfl);
      st->last_mu = mu;
      st->lam *= mu;
      st->prev_ovfl = st->ovfl;
      st->best_flag = 0;
      st->it += 1;
      if (st->it >= gp.max_iters) {
        st->done = 1;
      } else {
        st->gamma = gp.gamma_tab[st->it];
      }
      st->lam_eval = st->lam;
    }
  }
}

// ---------------------------------------------------------------------------
// host launchers
// ---------------------------------------------------------------------------
// K2 of the loop: spatially sorted, shared-memory privatised scatter of the
// cells / fillers + per-macro tiles, into gp.rho_fx (int64 fixed point)
#ifndef P3D_RESORT_EVERY
#define P3D_RESORT_EVERY 8
#endif
static void scatter_k2(const p3d_gp& gp, const int* halt, cudaStream_t s) {
  CloudGP cl;
  cl.pos = gp.v;
  cl.n_inst = gp.n_inst;
  cl.n_obj = gp.n_obj;
  cl.wt = gp.w_top; cl.ht = gp.h_top; cl.wb = gp.w_bot; cl.hb = gp.h_bot;
  cl.fw = gp.fill_w; cl.fh = gp.fill_h;
  cl.macro = gp.is_macro;
  cl.dz = gp.grid.dz;
  cl.target_density = gp.target_density;
#ifndef P3D_SCATTER_POS4
#define P3D_SCATTER_POS4 1
#endif
#if P3D_SCATTER_POS4
  // inside the loop (halt set) K5 / gp_init / gp_evaluate keep pos4 (evict-last)
  // in step with v for the instances, as K1 relies on too; the sorted scatter
  // then reads a cell's centre from it in one sector.  The per-op density
  // call (halt null) reads v only.
  if (halt && gp.pos4) cl.pos4 = reinterpret_cast<const double4*>(gp.pos4);
#endif
  if (gp.ts_order) {
    TileSort ts;
    ts.n_tiles = gp.ts_n_tiles;
    ts.tiles_x = gp.ts_tiles_x;
    ts.tiles_y = gp.ts_tiles_y;
    ts.margin = gp.ts_margin;
    ts.tile_of = gp.ts_tile_of;
    ts.hist = gp.ts_hist;
    ts.start = gp.ts_start;
    ts.cursor = gp.ts_cursor;
    ts.order = gp.ts_order;
    ts.rec = gp.ts_rec;
    ts.counter = &gp.st->counters[kCntTile];
    ts.i0 = gp.sh_i0;
    ts.ni = gp.sh_i1 - gp.sh_i0;
    ts.f0 = gp.sh_f0;
    // ts_order holds [n_obj] tiles, then [n_obj] perm, then the valid flag and
    // the iteration's sort decision
    ts.perm = gp.ts_order + gp.n_obj;
    ts.valid = gp.ts_order + 2 * (long long)gp.n_obj;
    ts.decision = ts.valid + 1;
    ts.it = &gp.st->it;
    ts.every = P3D_RESORT_EVERY;
    launch_scatter_tiled(cl, own_count(gp), gp.n_macro, gp.macro_ids, gp.grid, ts, gp.rho_fx,
                         halt, s);
  } else {
    launch_scatter(cl, gp.n_obj, gp.n_macro, gp.macro_ids, gp.grid, gp.rho_fx, halt, s);
  }
}

// ---- the stages of one evaluation (shared by the fused and sharded loops)
static void launch_k1(const p3d_gp& gp, cudaStream_t s) {
  p3d_loop_state* st = gp.st;
  const int* halt = &st->done;
  double* finals = gp.partials + (long long)kSlotFinal * kPartialStride;
  // K1 (degree-bucketed, register-resident nets)
  FusedNetArgs na{};
  na.n_net = gp.topo.n_net;
  na.n_tasks = gp.f_n_tasks;
  // shard_size 0: the fused loop; halo mode: this rank's own task list
  const bool rr = gp.shard_size > 0 && !gp.shard_halo;
  na.task_rank = rr ? gp.shard_rank : 0;
  na.task_size = rr ? gp.shard_size : 1;
  na.tasks = reinterpret_cast<const int4*>(gp.f_tasks);
  na.task_t0 = gp.f_task_t0;
  na.n_generic = gp.f_n_generic;
  na.generic_nets = gp.f_generic_nets;
  na.gpartials = gp.partials + (long long)kSlotGeneric * kPartialStride;
  na.gcounter = &st->counters[kCntGeneric];
  na.generic6 = finals + kFinGeneric;
  na.blocks = gp.nblk_net;
  na.net_base = gp.f_net_base;
  na.net_deg = gp.f_net_deg;
  na.net_stride = gp.f_net_stride;
  na.net_dup = gp.f_net_dup;
  na.pin_inst = gp.f_pin_inst;
  na.slot = gp.f_pin_slot;
  na.off = reinterpret_cast<const float4*>(gp.f_pin_off);
  na.pos4 = reinterpret_cast<const double4*>(gp.pos4);
  na.dz2 = gp.grid.dz / 2;
  na.gamma_ptr = &st->gamma;
  na.scale4 = 4.0 / gp.grid.dz;
  na.out_f = reinterpret_cast<float4*>(gp.pin_out_f);
  na.out_fd = gp.pin_out_fd;
  na.out_d = gp.wl_f32 ? nullptr : gp.pin_out;
  na.partials = gp.partials + (long long)kSlotNet * kPartialStride;
  na.counter = &st->counters[kCntNet];
  na.final6 = gp.shard_size > 0 ? gp.shard_tot : finals + kFinNet;  // sharded: local totals
  na.halt = halt;
  if (na.n_net > 0) launch_fused_net(na, gp.wl_f32 != 0, s);
}

static void launch_k1b(const p3d_gp& gp, cudaStream_t s) {
  p3d_loop_state* st = gp.st;
  const int* halt = &st->done;
  double* finals = gp.partials + (long long)kSlotFinal * kPartialStride;
  // K1b owner gather (per-instance sums; L1 norms + Eq. 17 scale on one GPU)
  FusedGatherArgs ga{};
  ga.n_obj = gp.n_inst;
  ga.obj0 = 0;
  if (gp.shard_size > 0 && gp.shard_halo) {  // own slab only (complete: every net touching it ran here)
    ga.obj0 = gp.sh_i0;
    ga.n_obj = gp.sh_i1 - gp.sh_i0;
  }
  // 8 CTAs per SM of a B200 as a constant (the block count partitions the
  // norms' ordered sums, like gp.GRID_SMS): measured +0.5% over 2,048 CTAs
  // and +0.2% over 592 (late round 2, three A/B rounds)
  static const int gather_cap = std::max(1, std::min(kMaxBlocks, getenv("P3D_NBLK_GATHER") ? atoi(getenv("P3D_NBLK_GATHER")) : 8 * 148));
  ga.blocks = grid_blocks(ga.n_obj, 256, gather_cap);
  ga.obj_slot_ptr = gp.topo.obj_slot_ptr;
  ga.in_f = reinterpret_cast<const float4*>(gp.pin_out_f);
  ga.in_fd = gp.pin_out_fd;
  ga.in_d = gp.wl_f32 ? nullptr : gp.pin_out;
  ga.out = gp.inst_g;
  ga.partials = gp.partials + (long long)kSlotGather * kPartialStride;
  ga.counter = &st->counters[kCntGather];
  ga.final_norms = gp.shard_size > 0 ? nullptr : finals + kFinNorm;  // sharded: NORMS stage
  ga.halt = halt;
  if (ga.n_obj > 0) launch_fused_gather(ga, s);
}

static int launch_k3(const p3d_gp& gp, cudaStream_t s) {
  p3d_loop_state* st = gp.st;
  const int* halt = &st->done;
  double* finals = gp.partials + (long long)kSlotFinal * kPartialStride;
  // K3 (+ overflow, re-zero)
  SpecOvfl ov;
  ov.zero = 1;
  ov.rho_t_fx = gp.rho_t_fx;
  ov.partials = gp.partials + (long long)kSlotOvfl * kPartialStride;
  ov.counter = &st->counters[kCntOvfl];
  ov.out = finals + kFinOvfl;
  // the int64 excess total: the (otherwise unused) last double of the slot
  ov.acc = reinterpret_cast<unsigned long long*>(ov.partials + kPartialStride - 1);
  ov.scale = gp.movable_volume > 0 ? 9.094947017729282379150390625e-13 * gp.grid.bin_vol / gp.movable_volume : 0.0;
  const int rc = launch_spectral_ex(&gp.grid, nullptr, gp.rho_fx, nullptr, nullptr, gp.maps,
                                    gp.spec_scratch, halt, &ov, s);
  if (rc) return rc;
  return 0;
}

static int eval_kernels(const p3d_gp& gp, cudaStream_t s, cudaEvent_t* ev = nullptr,
                        bool external = false) {
  auto mark = [&](int k) {
    if (!ev) return;
    if (external) cudaEventRecordWithFlags(ev[k], s, cudaEventRecordExternal);
    else cudaEventRecord(ev[k], s);
  };
  mark(0);
  launch_k1(gp, s);
  mark(1);
  launch_k1b(gp, s);
  mark(2);
  scatter_k2(gp, &gp.st->done, s);  // K2
  mark(3);
  if (const int rc = launch_k3(gp, s)) return rc;  // K3 (+ overflow, re-zero)
  mark(4);
  pdl_launch_tag(16, dens_kernel, gp.n_macro + gp.nblk_dens, 256, 0, s, gp);  // K4
  mark(5);
  return check_launch("gp evaluation kernels");
}

// The WL branch (K1, K1b) and the density branch (K2, K3) are independent
// until K4: with gp.overlap the density branch forks onto a high-priority
// side stream (its latency-bound kernels get SM slots as soon as they free
// up, next to the persistent K1 wave) and joins before K4; graph capture turns
// this into two concurrent branches.
struct ForkJoin {
  cudaStream_t side = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
};
static ForkJoin& fork_join() {  // one side stream + events per device
  static ForkJoin f[kMaxDevices];
  return f[current_device()];
}
static void overlap_setup() {  // outside any capture (gp_init / gp_evaluate)
  ForkJoin& f = fork_join();
  if (f.side) return;
  int least = 0, greatest = 0;
  cudaDeviceGetStreamPriorityRange(&least, &greatest);
  const char* e = getenv("P3D_OVERLAP_PRIO");
  const int prio = (e && e[0] == '0') ? least : greatest;
  cudaStreamCreateWithPriority(&f.side, cudaStreamNonBlocking, prio);
  cudaEventCreateWithFlags(&f.fork, cudaEventDisableTiming);
  cudaEventCreateWithFlags(&f.join, cudaEventDisableTiming);
}

// timing probe only (results are wrong): P3D_PROBE_SKIP bitmask drops K1 (1),
// K1b (2), K2 (4) or K3 (8) from the overlapped iteration, to read each
// stage's share of the critical path off the bench
static int probe_skip() {
  static const int v = getenv("P3D_PROBE_SKIP") ? atoi(getenv("P3D_PROBE_SKIP")) : 0;
  return v;
}

static int eval_kernels_overlap(const p3d_gp& gp, cudaStream_t s) {
  ForkJoin& f = fork_join();
  if (!f.side) return eval_kernels(gp, s);
  const int skip = probe_skip();
  cudaEventRecord(f.fork, s);
  cudaStreamWaitEvent(f.side, f.fork, 0);
  if (!(skip & 4)) scatter_k2(gp, &gp.st->done, f.side);
  if (!(skip & 8))
    if (const int rc = launch_k3(gp, f.side)) return rc;
  if (!(skip & 1)) launch_k1(gp, s);
  if (!(skip & 2)) launch_k1b(gp, s);
  cudaEventRecord(f.join, f.side);
  cudaStreamWaitEvent(s, f.join, 0);
  pdl_launch_tag(16, dens_kernel, gp.n_macro + gp.nblk_dens, 256, 0, s, gp);
  return check_launch("gp evaluation kernels (overlapped)");
}

int gp_iterate(const p3d_gp& gp, cudaStream_t s, bool steady) {
  if (const int rc = gp.overlap ? eval_kernels_overlap(gp, s) : eval_kernels(gp, s)) return rc;
  if (!steady) pdl_launch_tag(32, gmax0_kernel, gp.nblk_obj, 256, 0, s, gp);
  pdl_launch_tag(64, advance_kernel, gp.nblk_obj, 256, 0, s, gp);
  return check_launch("gp_iterate");
}

// Same launches with an event between stages (host-synchronising; used by the
// benchmark to attribute iteration time to K1..K5, never inside a graph).
int gp_iterate_profiled(const p3d_gp& gp, cudaStream_t s, float* ms) {
  static cudaEvent_t ev[8] = {nullptr};
  if (!ev[0])
    for (int k = 0; k < 8; ++k) cudaEventCreate(&ev[k]);
  if (const int rc = eval_kernels(gp, s, ev)) return rc;
  pdl_launch_tag(32, gmax0_kernel, gp.nblk_obj, 256, 0, s, gp);
  cudaEventRecord(ev[6], s);
  pdl_launch_tag(64, advance_kernel, gp.nblk_obj, 256, 0, s, gp);
  cudaEventRecord(ev[7], s);
  cudaEventSynchronize(ev[7]);
  for (int k = 0; k < 7; ++k) cudaEventElapsedTime(&ms[k], ev[k], ev[k + 1]);
  return check_launch("gp_iterate_profiled");
}

// Capturable variant: the stage events become event-record nodes of a CUDA
// graph, so a replayed graph is attributed without host gaps; read the stage
// times with gp_stage_times after the replay completes.
static cudaEvent_t g_marks[8] = {nullptr};

int gp_iterate_marked(const p3d_gp& gp, cudaStream_t s) {
  if (!g_marks[0])
    for (int k = 0; k < 8; ++k) cudaEventCreate(&g_marks[k]);
  if (const int rc = eval_kernels(gp, s, g_marks, true)) return rc;
  pdl_launch_tag(32, gmax0_kernel, gp.nblk_obj, 256, 0, s, gp);
  cudaEventRecordWithFlags(g_marks[6], s, cudaEventRecordExternal);
  pdl_launch_tag(64, advance_kernel, gp.nblk_obj, 256, 0, s, gp);
  cudaEventRecordWithFlags(g_marks[7], s, cudaEventRecordExternal);
  return check_launch("gp_iterate_marked");
}

// The overlapped iteration with event-record nodes at the branch points
// (graph-capturable): t[k] = ms from the fork to mark k, k = 1 K1 net done,
// 2 K1b done (WL branch), 3 K2 done, 4 K3 done (density branch), 5 K4 done,
// 6 K5a done, 7 K5b done -- the iteration's critical path as it runs
// (the per-stage times above are taken on the serialised variant).
static cudaEvent_t g_omarks[8] = {nullptr};

int gp_iterate_marked_overlap(const p3d_gp& gp, cudaStream_t s) {
  if (!g_omarks[0])
    for (int k = 0; k < 8; ++k) cudaEventCreate(&g_omarks[k]);
  ForkJoin& f = fork_join();
  if (!f.side) return P3D_ERR_ARG;
  auto mark = [&](int k, cudaStream_t st) { cudaEventRecordWithFlags(g_omarks[k], st, cudaEventRecordExternal); };
  mark(0, s);
  cudaEventRecord(f.fork, s);
  cudaStreamWaitEvent(f.side, f.fork, 0);
  scatter_k2(gp, &gp.st->done, f.side);
  mark(3, f.side);
  if (const int rc = launch_k3(gp, f.side)) return rc;
  mark(4, f.side);
  launch_k1(gp, s);
  mark(1, s);
  launch_k1b(gp, s);
  mark(2, s);
  cudaEventRecord(f.join, f.side);
  cudaStreamWaitEvent(s, f.join, 0);
  pdl_launch_tag(16, dens_kernel, gp.n_macro + gp.nblk_dens, 256, 0, s, gp);
  mark(5, s);
  pdl_launch_tag(32, gmax0_kernel, gp.nblk_obj, 256, 0, s, gp);
  mark(6, s);
  pdl_launch_tag(64, advance_kernel, gp.nblk_obj, 256, 0, s, gp);
  mark(7, s);
  return check_launch("gp_iterate_marked_overlap");
}

int gp_overlap_times(float* t) {
  if (!g_omarks[0]) return P3D_ERR_ARG;
  if (cudaEventSynchronize(g_omarks[7]) != cudaSuccess) return check_launch("overlap times");
  for (int k = 1; k < 8; ++k) cudaEventElapsedTime(&t[k - 1], g_omarks[0], g_omarks[k]);
  return check_launch("overlap times");
}

int gp_stage_times(float* ms) {
  if (!g_marks[0]) return P3D_ERR_ARG;
  if (cudaEventSynchronize(g_marks[7]) != cudaSuccess) return check_launch("stage times");
  for (int k = 0; k < 7; ++k) cudaEventElapsedTime(&ms[k], g_marks[k], g_marks[k + 1]);
  return check_launch("stage times");
}

// kernels enqueued by one gp_iterate (for the benchmark's launch count)
int gp_kernels_per_iteration(const p3d_gp& gp) {
  const int k2 = gp.ts_order ? 3 /*histogram+scan+macros, place, scatter*/
                             : 1 + (gp.n_macro > 0) /*cells, macros*/;
  return (gp.topo.n_net > 0) + (gp.f_n_generic > 0) /*net*/ + (gp.n_inst > 0) /*gather*/ + k2 +
         (spectral_fast_ok(&gp.grid) ? 3 : 6) /*spectral*/ +
         1 /*dens*/ + 2 /*step, advance*/;
}

int gp_evaluate(const p3d_gp& gp, double lam, double gamma, cudaStream_t s) {
  overlap_setup();
  spectral_setup();
  tiled_scatter_setup();
  fused_net_setup();
  eval_setup_kernel<<<1, 1, 0, s>>>(gp, lam, gamma);
  if (gp.n_inst > 0)
    pos4_kernel<<<grid_blocks(gp.n_inst, 256, 4096), 256, 0, s>>>(gp.n_inst, gp.n_obj, gp.v, gp.pos4);
  if (const int rc = eval_kernels(gp, s)) return rc;
  return check_launch("gp_evaluate");
}

int gp_init(const p3d_gp& gp, const double* pos0, cudaStream_t s) {
  overlap_setup();
  spectral_setup();
  tiled_scatter_setup();
  fused_net_setup();
  init_state_kernel<<<1, 1, 0, s>>>(gp);
  const int b = grid_blocks(gp.n_obj, 256, 4096);
  project_kernel<<<b, 256, 0, s>>>(gp, pos0, gp.u);
  copy3_kernel<<<b, 256, 0, s>>>(gp.n_obj, gp.u, gp.v, gp.best);
  if (gp.n_inst > 0)
    pos4_kernel<<<grid_blocks(gp.n_inst, 256, 4096), 256, 0, s>>>(gp.n_inst, gp.n_obj, gp.v, gp.pos4);
  cudaMemsetAsync(gp.rho_fx, 0, sizeof(int64_t) * (size_t)gp.grid.nx * gp.grid.ny * gp.grid.nz, s);
  return check_launch("gp_init");
}

// ---------------------------------------------------------------------------
// sharded loop (config 4): the stages that follow a collective
// ---------------------------------------------------------------------------
// L1 norms of this rank's instance slab of the reduced owner sums (partials
// into shard_tot[20, 23), all-reduced by the host, then norms_final_kernel)
__global__ void __launch_bounds__(256) inst_norms_kernel(p3d_gp gp) {
  if (gp.st->done) return;
  __shared__ double red[32 * 3];
  double acc[3] = {0, 0, 0};
  const double4* g4 = reinterpret_cast<const double4*>(gp.inst_g);
  for (int i = gp.sh_i0 + blockIdx.x * blockDim.x + threadIdx.x; i < gp.sh_i1;
       i += gridDim.x * blockDim.x) {
    const double4 g = g4[i];
    acc[0] += fabs(g.x);
    acc[1] += fabs(g.y);
    acc[2] += fabs(g.w);
  }
  double* part = gp.partials + (long long)kSlotGather * kPartialStride;
  block_sum<3>(acc, red);
  if (threadIdx.x == 0)
    for (int q = 0; q < 3; ++q) part[q * gridDim.x + blockIdx.x] = acc[q];
  if (last_block(&gp.st->counters[kCntGather])) {
    double n[3];
    ordered_sums<3>(part, gridDim.x, gridDim.x, red, n);
    if (threadIdx.x == 0)
      for (int q = 0; q < 3; ++q) gp.shard_tot[20 + q] = n[q];
  }
}

// the norms over all ranks + the Eq. 17 scale (identical on every rank)
__global__ void norms_final_kernel(p3d_gp gp) {
  if (gp.st->done) return;
  double* f = fin(gp) + kFinNorm;
  const double* t = gp.shard_tot + 20;
  f[0] = t[0];
  f[1] = t[1];
  f[2] = t[2];
  f[3] = t[2] == 0.0 ? 0.0 : (t[0] + t[1]) / (2.0 * t[2]);  // Eq. 17
}

// loop control with the all-reduced totals (net: shard_tot[0,6), density:
// shard_tot[8,14), the last step's |v - v_prev|^2: shard_tot[14]); identical
// on every rank
__global__ void shard_control_kernel(p3d_gp gp) {
  if (gp.st->done) return;
  double* f = fin(gp);
  const double* t = gp.shard_tot;
  for (int q = 0; q < 6; ++q) f[kFinNet + q] = t[q];
  gp.st->dv2_next = t[14];  // |v - v_prev|^2 summed over the ranks' objects
  control_after_eval(gp, t[8], t[9], t[10], t[11], t[12], t[13]);
}

// iteration 0: the initial step from the max over ranks of |g| (gp.py:198-202)
__global__ void step0_control_kernel(p3d_gp gp) {
  p3d_loop_state* st = gp.st;
  if (st->done || st->step_set || st->stop_now) return;
  const double gm = gp.shard_tot[16];
  st->gmax = gm;
  st->step = gm == 0.0 ? 1.0 : gp.step_scale / gm;
  st->step_set = 1;
  step_tail(gp);
}

int gp_shard_stage(const p3d_gp& gp, int stage, cudaStream_t s) {
  spectral_setup();
  tiled_scatter_setup();
  fused_net_setup();
  switch (stage) {
    case P3D_SH_NET: if (gp.topo.n_net > 0) launch_k1(gp, s); break;
    case P3D_SH_GATHER: if (gp.n_inst > 0) launch_k1b(gp, s); break;
    case P3D_SH_NORMS:
      inst_norms_kernel<<<grid_blocks(gp.n_inst, 256, kMaxBlocks), 256, 0, s>>>(gp);
      break;
    case P3D_SH_NORMS_FINAL: norms_final_kernel<<<1, 1, 0, s>>>(gp); break;
    case P3D_SH_SCATTER: scatter_k2(gp, &gp.st->done, s); break;
    case P3D_SH_SPECTRAL: if (const int rc = launch_k3(gp, s)) return rc; break;
    case P3D_SH_DENS: pdl_launch_tag(16, dens_kernel, gp.n_macro + gp.nblk_dens, 256, 0, s, gp); break;
    case P3D_SH_CONTROL: shard_control_kernel<<<1, 1, 0, s>>>(gp); break;
    case P3D_SH_STEP0: pdl_launch_tag(32, gmax0_kernel, gp.nblk_obj, 256, 0, s, gp); break;
    case P3D_SH_STEP0_CONTROL: step0_control_kernel<<<1, 1, 0, s>>>(gp); break;
    case P3D_SH_ADVANCE: pdl_launch_tag(64, advance_kernel, gp.nblk_obj, 256, 0, s, gp); break;
    default: return P3D_ERR_ARG;
  }
  return check_launch("gp_shard_stage");
}

int gp_density_fx(const p3d_gp& gp, int64_t* out, cudaStream_t s) {
  tiled_scatter_setup();
  const size_t bytes = sizeof(int64_t) * (size_t)gp.grid.nx * gp.grid.ny * gp.grid.nz;
  cudaMemsetAsync(gp.rho_fx, 0, bytes, s);
  scatter_k2(gp, nullptr, s);
  cudaMemcpyAsync(out, gp.rho_fx, bytes, cudaMemcpyDeviceToDevice, s);
  cudaMemsetAsync(gp.rho_fx, 0, bytes, s);
  return check_launch("gp_density_fx");
}

int gp_project(const p3d_gp& gp, const double* in, double* out, cudaStream_t s) {
  project_kernel<<<grid_blocks(gp.n_obj, 256, 4096), 256, 0, s>>>(gp, in, out);
  return check_launch("gp_project");
}

}  // namespace p3d
