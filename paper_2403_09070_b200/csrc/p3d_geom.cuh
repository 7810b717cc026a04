// Charge geometry shared by the density scatter (K2) and gather (K4).
// Every expression mirrors numpy's operation order in density.py:134-196 so
// that, compiled with -fmad=false, the per-(object, bin) overlap volumes are
// bit-identical to the reference's _direct_terms.
#pragma once

#include "p3d_common.cuh"

namespace p3d {

struct Charge {
  double x, y, z, w, h, dep, weight;
};

// density.py:134-147 (Eqs. 6-7); z clamped to [dz/4, 3dz/4] first
__device__ __forceinline__ void dynamic_wh(double z, double dz, bool macro, double wt, double ht,
                                           double wb, double hb, double& w, double& h) {
  const double zc = clipd(z, dz / 4, 3 * dz / 4);
  if (macro) {
    const double t = 2 * zc / dz - 0.5;
    w = t * wt + (1 - t) * wb;
    h = t * ht + (1 - t) * hb;
  } else {
    const bool top = (zc - dz / 2) > 0.0;
    w = top ? wt : wb;
    h = top ? ht : hb;
  }
}

struct AxisSpan {
  double lo, hi;
  int i0, i1;
};

// density.py:155-169: clipped extent and inclusive bin range on one axis
// (ystep = 1 / step: both quotients from one reciprocal, same values as lo /
// step and hi / step, see div_rcp)
__device__ __forceinline__ AxisSpan axis_span(double c, double size, double extent, double step,
                                              double ystep, int n) {
  AxisSpan s;
  s.lo = clipd(c - size / 2, 0.0, extent);
  s.hi = clipd(c + size / 2, 0.0, extent);
  long long a = (long long)floor(div_rcp(s.lo, step, ystep));
  long long b = (long long)ceil(div_rcp(s.hi, step, ystep)) - 1;
  a = a < 0 ? 0 : (a > n - 1 ? n - 1 : a);
  b = b < 0 ? 0 : (b > n - 1 ? n - 1 : b);
  if (b < a) b = a;
  s.i0 = (int)a;
  s.i1 = (int)b;
  return s;
}

// density.py:172-173
__device__ __forceinline__ double overlap_len(const AxisSpan& s, int i, double step) {
  return dmax(dmin(s.hi, (double)(i + 1) * step) - dmax(s.lo, (double)i * step), 0.0);
}

// overlap_len of the first M bins of a span at once, entries k >= nr zero.
// The reference's min/max are kept only where they can bind: with
// i0 = floor(lo / step) and i1 = ceil(hi / step) - 1 (rounded quotients,
// monotone rounding) every interior boundary e_k = (i0 + k) * step satisfies
// lo <= e_k for k >= 1 and e_k <= hi for i0 + k <= i1, so
// max(lo, e_k) = e_k, min(hi, e_k+1) = e_k+1 and the clip at 0 is the
// identity there: the values are identical to overlap_len's.
#ifndef P3D_AXIS_WEIGHTS
#define P3D_AXIS_WEIGHTS 1
#endif
template <int M>
__device__ __forceinline__ void axis_weights(const AxisSpan& s, double step, double (&w)[M]) {
  const int nr = s.i1 - s.i0 + 1;
#if P3D_AXIS_WEIGHTS
  const double d0 = (double)s.i0;
  double e[M + 1];
#pragma unroll
  for (int k = 0; k <= M; ++k) e[k] = (d0 + (double)k) * step;  // == (double)(i0 + k) * step
  double right_edge = e[M];
#pragma unroll
  for (int k = 1; k < M; ++k)
    if (nr == k) right_edge = e[k];
  right_edge = dmin(s.hi, right_edge);
#pragma unroll
  for (int k = 0; k < M; ++k) {
    const double right = (k == nr - 1) ? right_edge : e[k + 1];
    const double v = k == 0 ? dmax(right - dmax(s.lo, e[0]), 0.0) : right - e[k];
    w[k] = k < nr ? v : 0.0;
  }
#else
#pragma unroll
  for (int k = 0; k < M; ++k) w[k] = k < nr ? overlap_len(s, s.i0 + k, step) : 0.0;
#endif
}

struct Footprint {
  AxisSpan ax, ay, az;
};

__device__ __forceinline__ Footprint footprint(const Charge& c, const p3d_grid& g) {
  Footprint f;
  f.ax = axis_span(c.x, c.w, g.dx, g.wb, 1.0 / g.wb, g.nx);
  f.ay = axis_span(c.y, c.h, g.dy, g.hb, 1.0 / g.hb, g.ny);
  f.az = axis_span(c.z, c.dep, g.dz, g.db, 1.0 / g.db, g.nz);
  return f;
}

// ---------------------------------------------------------------------------
// charge sources
// ---------------------------------------------------------------------------
struct CloudArrays {  // explicit ChargeCloud (per-op API)
  p3d_cloud c;
  __device__ __forceinline__ bool is_macro(int i) const { return c.is_macro && c.is_macro[i]; }
  __device__ __forceinline__ double cx(int i) const { return c.x[i]; }
  __device__ __forceinline__ double cy(int i) const { return c.y[i]; }
  __device__ __forceinline__ Charge get(int i) const {
    Charge q;
    q.x = c.x[i]; q.y = c.y[i]; q.z = c.z[i];
    q.w = c.w[i]; q.h = c.h[i]; q.dep = c.dep[i]; q.weight = c.weight[i];
    return q;
  }
};

struct CloudGP {  // Gp3dProblem.cloud(pos) computed on the fly (gp.py:267-278)
  const double* pos;  // [3][n_obj]
  int n_inst, n_obj;
  const double *wt, *ht, *wb, *hb, *fw, *fh;
  const uint8_t* macro;
  double dz, target_density;
  const double4* pos4 = nullptr;  // optional [n_inst] AoS copy of pos (x, y, z, 0)
  __device__ __forceinline__ bool is_macro(int i) const { return i < n_inst && macro[i]; }
  __device__ __forceinline__ double cx(int i) const { return pos[i]; }
  __device__ __forceinline__ double cy(int i) const { return pos[n_obj + i]; }
  __device__ __forceinline__ Charge get(int i) const {
    Charge q;
    q.x = pos[i];
    q.y = pos[n_obj + i];
    q.z = pos[2 * n_obj + i];
    if (i < n_inst) {
      const bool m = macro[i] != 0;
      dynamic_wh(q.z, dz, m, wt[i], ht[i], wb[i], hb[i], q.w, q.h);
      q.weight = m ? target_density : 1.0;
    } else {
      q.w = fw[i - n_inst];
      q.h = fh[i - n_inst];
      q.weight = 1.0;
    }
    q.dep = dz / 2;
    return q;
  }
  // get(i) for an object known not to be a macro (the scatter's sorted cells
  // and fillers): the same values, loading only the die's width / height pair
  // get_nonmacro with the sizes given: (wt, ht), (wb, hb) of an instance,
  // (fw, fh) twice for a filler
  __device__ __forceinline__ Charge get_sized(int i, double2 s_top, double2 s_bot) const {
    Charge q;
    if (pos4 && i < n_inst) {
      const double4 p = pos4[i];
      q.x = p.x; q.y = p.y; q.z = p.z;
    } else {
      q.x = pos[i];
      q.y = pos[n_obj + i];
      q.z = pos[2 * n_obj + i];
    }
    const double zc = clipd(q.z, dz / 4, 3 * dz / 4);  // dynamic_wh's cell branch
    const bool top = (i >= n_inst) || (zc - dz / 2) > 0.0;
    q.w = top ? s_top.x : s_bot.x;
    q.h = top ? s_top.y : s_bot.y;
    q.weight = 1.0;
    q.dep = dz / 2;
    return q;
  }
  __device__ __forceinline__ Charge get_nonmacro(int i) const {
    Charge q;
    if (pos4 && i < n_inst) {  // one 32-byte load instead of three scattered ones
      const double4 p = pos4[i];
      q.x = p.x; q.y = p.y; q.z = p.z;
    } else {
      q.x = pos[i];
      q.y = pos[n_obj + i];
      q.z = pos[2 * n_obj + i];
    }
    if (i < n_inst) {
      const double zc = clipd(q.z, dz / 4, 3 * dz / 4);  // dynamic_wh's cell branch
      const bool top = (zc - dz / 2) > 0.0;
      const double* pw = top ? wt : wb;
      const double* ph = top ? ht : hb;
      q.w = pw[i];
      q.h = ph[i];
    } else {
      q.w = fw[i - n_inst];
      q.h = fh[i - n_inst];
    }
    q.weight = 1.0;
    q.dep = dz / 2;
    return q;
  }
};

__device__ __forceinline__ double charge_of(const Charge& q) {
  return q.weight * (q.w * q.h * q.dep);  // ChargeCloud.charge (density.py:71-77)
}

// ---------------------------------------------------------------------------
// K2: fixed-point scatter of one object's overlaps (thread-serial)
// ---------------------------------------------------------------------------
__device__ __forceinline__ void scatter_object(const Charge& q, const p3d_grid& g,
                                               unsigned long long* rho) {
  const Footprint f = footprint(q, g);
  for (int ix = f.ax.i0; ix <= f.ax.i1; ++ix) {
    const double wx = overlap_len(f.ax, ix, g.wb);
    for (int iy = f.ay.i0; iy <= f.ay.i1; ++iy) {
      const double wxy = wx * overlap_len(f.ay, iy, g.hb);
      for (int iz = f.az.i0; iz <= f.az.i1; ++iz) {
        const double vol = wxy * overlap_len(f.az, iz, g.db);
        const long long t = __double2ll_rn((q.weight * vol) * g.fx_scale);
        if (t) atomicAdd(rho + ((long long)(ix * g.ny + iy) * g.nz + iz), (unsigned long long)t);
      }
    }
  }
}

// block-cooperative scatter of one large object (per-macro tile path)
__device__ __forceinline__ void scatter_object_block(const Charge& q, const p3d_grid& g,
                                                     unsigned long long* rho, int part = 0,
                                                     int nparts = 1) {
  const Footprint f = footprint(q, g);
  const int nxr = f.ax.i1 - f.ax.i0 + 1, nyr = f.ay.i1 - f.ay.i0 + 1, nzr = f.az.i1 - f.az.i0 + 1;
  const int tot = nxr * nyr * nzr;
  for (int t = part * blockDim.x + threadIdx.x; t < tot; t += nparts * blockDim.x) {
    const int iz = f.az.i0 + t % nzr;
    const int iy = f.ay.i0 + (t / nzr) % nyr;
    const int ix = f.ax.i0 + t / (nzr * nyr);
    const double wxy = overlap_len(f.ax, ix, g.wb) * overlap_len(f.ay, iy, g.hb);
    const double vol = wxy * overlap_len(f.az, iz, g.db);
    const long long v = __double2ll_rn((q.weight * vol) * g.fx_scale);
    if (v) atomicAdd(rho + ((long long)(ix * g.ny + iy) * g.nz + iz), (unsigned long long)v);
  }
}

// ---------------------------------------------------------------------------
// K4: overlap-weighted means of the 4 interleaved maps (density.py:376-386)
// ---------------------------------------------------------------------------
__device__ __forceinline__ void gather_generic(const Footprint& f, const p3d_grid& g,
                                               const double4* m4, double& tot, double (&a)[4]) {
  for (int ix = f.ax.i0; ix <= f.ax.i1; ++ix) {
    const double wx = overlap_len(f.ax, ix, g.wb);
    for (int iy = f.ay.i0; iy <= f.ay.i1; ++iy) {
      const double wxy = wx * overlap_len(f.ay, iy, g.hb);
      for (int iz = f.az.i0; iz <= f.az.i1; ++iz) {
        const double vol = wxy * overlap_len(f.az, iz, g.db);
        const double4 m = m4[(long long)(ix * g.ny + iy) * g.nz + iz];
        tot += vol;
        a[0] += m.x * vol;
        a[1] += m.y * vol;
        a[2] += m.z * vol;
        a[3] += m.w * vol;
      }
    }
  }
}

// Footprints of at most MX x MY x MZ bins (every standard cell and filler of
// the BASELINE configs): per-axis overlap lengths computed once, the bin loop
// fully unrolled with guards so all map loads are in flight together.  Same
// terms, same accumulation order as gather_generic.
template <int MX, int MY, int MZ>
__device__ __forceinline__ void gather_small(const Footprint& f, const p3d_grid& g,
                                             const double4* m4, double& tot, double (&a)[4]) {
  const int nxr = f.ax.i1 - f.ax.i0 + 1, nyr = f.ay.i1 - f.ay.i0 + 1, nzr = f.az.i1 - f.az.i0 + 1;
  double wx[MX], wy[MY], wz[MZ];
  axis_weights<MX>(f.ax, g.wb, wx);
  axis_weights<MY>(f.ay, g.hb, wy);
  axis_weights<MZ>(f.az, g.db, wz);
  const long long b0 = (long long)(f.ax.i0 * g.ny + f.ay.i0) * g.nz + f.az.i0;
#pragma unroll
  for (int x = 0; x < MX; ++x) {
#pragma unroll
    for (int y = 0; y < MY; ++y) {
      const double wxy = wx[x] * wy[y];
#pragma unroll
      for (int z = 0; z < MZ; ++z) {
        if (x < nxr && y < nyr && z < nzr) {
          const double vol = wxy * wz[z];
          const double4 m = m4[b0 + ((long long)x * g.ny + y) * g.nz + z];
          tot += vol;
          a[0] += m.x * vol;
          a[1] += m.y * vol;
          a[2] += m.z * vol;
          a[3] += m.w * vol;
        }
      }
    }
  }
}

__device__ __forceinline__ void gather_object(const Charge& q, const p3d_grid& g,
                                              const double* maps, double (&mean)[4]) {
  const Footprint f = footprint(q, g);
  double tot = 0.0, a[4] = {0.0, 0.0, 0.0, 0.0};
  const double4* m4 = reinterpret_cast<const double4*>(maps);
#ifndef P3D_SMALL2
#define P3D_SMALL2 1
#endif
#if P3D_SMALL2
  // 2 x 2 x 2 first (every cell and filler of the BASELINE configs): the
  // unrolled 3 x 3 x 2 set issues its guarded-off slots too.  Same terms in
  // the same order, so the same sums.
  if (f.ax.i1 - f.ax.i0 < 2 && f.ay.i1 - f.ay.i0 < 2 && f.az.i1 - f.az.i0 < 2)
    gather_small<2, 2, 2>(f, g, m4, tot, a);
  else
#endif
  if (f.ax.i1 - f.ax.i0 < 3 && f.ay.i1 - f.ay.i0 < 3 && f.az.i1 - f.az.i0 < 2)
    gather_small<3, 3, 2>(f, g, m4, tot, a);
  else
    gather_generic(f, g, m4, tot, a);
  tot = dmax(tot, 1e-300);
  const double ytot = 1.0 / tot;
  mean[0] = div_rcp(a[0], tot, ytot);
  mean[1] = div_rcp(a[1], tot, ytot);
  mean[2] = div_rcp(a[2], tot, ytot);
  mean[3] = div_rcp(a[3], tot, ytot);
}

// block-cooperative macro means: sum m*vol over the footprint / unclipped
// volume (== the suffix-sum corner dots of density.py:489-530); thread 0 holds
// the result.
__device__ __forceinline__ void gather_object_block(const Charge& q, const p3d_grid& g,
                                                    const double* maps, double (&mean)[4],
                                                    double* red) {
  const Footprint f = footprint(q, g);
  const int nxr = f.ax.i1 - f.ax.i0 + 1, nyr = f.ay.i1 - f.ay.i0 + 1, nzr = f.az.i1 - f.az.i0 + 1;
  const int tot = nxr * nyr * nzr;
  const double4* m4 = reinterpret_cast<const double4*>(maps);
  double acc[4] = {0, 0, 0, 0};
  for (int t = threadIdx.x; t < tot; t += blockDim.x) {
    const int iz = f.az.i0 + t % nzr;
    const int iy = f.ay.i0 + (t / nzr) % nyr;
    const int ix = f.ax.i0 + t / (nzr * nyr);
    const double wxy = overlap_len(f.ax, ix, g.wb) * overlap_len(f.ay, iy, g.hb);
    const double vol = wxy * overlap_len(f.az, iz, g.db);
    const double4 m = m4[(long long)(ix * g.ny + iy) * g.nz + iz];
    acc[0] += m.x * vol;
    acc[1] += m.y * vol;
    acc[2] += m.z * vol;
    acc[3] += m.w * vol;
  }
  block_sum<4>(acc, red);
  const double vol = fmax(q.w * q.h * q.dep, 1e-300);
  mean[0] = acc[0] / vol;
  mean[1] = acc[1] / vol;
  mean[2] = acc[2] / vol;
  mean[3] = acc[3] / vol;
}

}  // namespace p3d
