// K1 — bistratal weighted-average wirelength, z-cut penalty, incremental
// finite-difference depth gradient, exact bistratal HPWL and crossing count.
//
// Reference: place3d/wirelength.py:76-98 (_segment_wa), 101-142 (NetBoxes),
// 167-198 (bistratal_spans, planar_objective, z_cut_penalty), 227-293
// (_axis_flip_delta, fd_z_gradient_incremental), gp.py:336-356 (exact WL,
// crossings).
//
// One thread owns one net (nets are processed in degree-grouped order so a
// warp's lanes run the same trip counts).  Per net it
//   pass 1  gathers pins and builds per-(net, die) first/second extrema with
//           multiplicity on x and y plus the z extent (NetBoxes, exact fp64);
//   pass 2  picks the branch per axis from the unsmoothed spans and forms the
//           WA exponential sums of that branch only (the other branch's value
//           and gradient are never used by planar_objective);
//   pass 3  writes per-pin gradients (x, y, cut-z) and the FD depth term.
// Per-pin results go to the pin's owner-sorted slot so the per-object sum
// (the reference's bincount) is an ordered, deterministic gather.
#include <stdio.h>

#include "p3d_common.cuh"
#include "p3d_internal.cuh"

namespace p3d {

struct Box {  // one axis, both dies
  int cnt[2];
  double hi1[2], hi2[2], lo1[2], lo2[2];
  __device__ __forceinline__ void init() {
#pragma unroll
    for (int d = 0; d < 2; ++d) {
      cnt[d] = 0;
      hi1[d] = hi2[d] = -P3D_INF;
      lo1[d] = lo2[d] = P3D_INF;
    }
  }
  // top-2 with multiplicity == sorted order statistics (wirelength.py:113-131)
  __device__ __forceinline__ void add(double c, int d) {
    cnt[d] += 1;
    if (c > hi1[d]) { hi2[d] = hi1[d]; hi1[d] = c; } else if (c > hi2[d]) { hi2[d] = c; }
    if (c < lo1[d]) { lo2[d] = lo1[d]; lo1[d] = c; } else if (c < lo2[d]) { lo2[d] = c; }
  }
  __device__ __forceinline__ double span(int d) const { return cnt[d] > 0 ? hi1[d] - lo1[d] : 0.0; }
  __device__ __forceinline__ double fmaxv() const { return fmax(hi1[0], hi1[1]); }
  __device__ __forceinline__ double fminv() const { return fmin(lo1[0], lo1[1]); }
  __device__ __forceinline__ double full() const {
    return (cnt[0] + cnt[1]) > 0 ? fmaxv() - fminv() : 0.0;
  }
  // wirelength.py:167-170
  __device__ __forceinline__ double bistratal() const { return fmax(full(), span(1) + span(0)); }
  // wirelength.py:227-248 (one pin flips die; pin offsets kept)
  __device__ __forceinline__ double flip_delta(double c, int d, double cur) const {
    const int o = 1 - d;
    double same = 0.0;
    if (cnt[d] > 1) {
      double nhi = (c == hi1[d]) ? hi2[d] : hi1[d];
      double nlo = (c == lo1[d]) ? lo2[d] : lo1[d];
      same = nhi - nlo;
    }
    double other = fmax(hi1[o], c) - fmin(lo1[o], c);
    return fmax(full(), same + other) - cur;
  }
};

struct WaSum {  // exponential sums of one segment
  double s1p, sxp, s1m, sxm;
  __device__ __forceinline__ void init() { s1p = sxp = s1m = sxm = 0.0; }
  __device__ __forceinline__ void add(double v, double hi, double lo, double inv_g) {
    double ep = exp((v - hi) / inv_g);
    double em = exp((lo - v) / inv_g);
    s1p += ep;
    sxp += v * ep;
    s1m += em;
    sxm += v * em;
  }
  __device__ __forceinline__ double vp() const { return sxp / s1p; }
  __device__ __forceinline__ double vm() const { return sxm / s1m; }
  __device__ __forceinline__ double value() const { return s1p > 0 ? vp() - vm() : 0.0; }
  // wirelength.py:94-96
  __device__ __forceinline__ double grad(double v, double hi, double lo, double gamma,
                                         double inv_g) const {
    double ep = exp((v - hi) / gamma);
    double em = exp((lo - v) / gamma);
    return ep / s1p * (1.0 + (v - vp()) / gamma) - em / s1m * (1.0 - (v - vm()) / gamma);
  }
};

// pins formed from instance centres + per-die offsets (wirelength.py:308-322)
struct PinsFromPos {
  const double* x;
  const double* y;
  const double* z;
  const double4* off;
  const int32_t* pin_inst;
  double dz2;
  __device__ __forceinline__ void get(int k, double& px, double& py, double& pz, int& top) const {
    int i = pin_inst[k];
    double zi = z[i];
    top = (zi - dz2) > 0.0;
    double4 o = off[k];
    px = x[i] + (top ? o.x : o.z);
    py = y[i] + (top ? o.y : o.w);
    pz = zi;
  }
};

// pins given directly (per-op API)
struct PinsDirect {
  const double* px;
  const double* py;
  const double* pz;
  const uint8_t* top;
  __device__ __forceinline__ void get(int k, double& x, double& y, double& z, int& t) const {
    x = px ? px[k] : 0.0;
    y = py ? py[k] : 0.0;
    z = pz ? pz[k] : 0.0;
    t = top ? (top[k] != 0) : 0;
  }
};

// exact bistratal extent of one axis with owner `w` forced to die `forced`
// (wirelength.py:145-150, 280-292); O(|P_e|)
template <class Pins>
__device__ double forced_bistratal(const Pins& pins, const int32_t* pin_inst, int p0, int p1,
                                   int w, int forced, int axis) {
  double thi = -P3D_INF, tlo = P3D_INF, bhi = -P3D_INF, blo = P3D_INF;
  double fhi = -P3D_INF, flo = P3D_INF;
  int nt = 0, nb = 0;
  for (int k = p0; k < p1; ++k) {
    double x, y, z;
    int t;
    pins.get(k, x, y, z, t);
    double c = axis == 0 ? x : y;
    if (pin_inst[k] == w) t = forced;
    fhi = fmax(fhi, c);
    flo = fmin(flo, c);
    if (t) { nt++; thi = fmax(thi, c); tlo = fmin(tlo, c); } else { nb++; bhi = fmax(bhi, c); blo = fmin(blo, c); }
  }
  double full = (p1 > p0) ? fhi - flo : 0.0;
  double st = nt ? thi - tlo : 0.0;
  double sb = nb ? bhi - blo : 0.0;
  return fmax(full, st + sb);
}

template <class Pins, bool PLANAR, bool CUT, bool FD>
__global__ void __launch_bounds__(256) net_kernel(NetArgs a, Pins pins) {
  if (a.halt && *a.halt) return;
  __shared__ double red[32 * 6];
  const double gamma = a.gamma_ptr ? *a.gamma_ptr : a.gamma;
  const double inv_g = gamma;  // (the sums divide by gamma like numpy)
  double acc[6] = {0, 0, 0, 0, 0, 0};  // planar x, planar y, cut, exact x, exact y, crossings
  const int stride = gridDim.x * blockDim.x;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < a.n_net; t += stride) {
    const int n = a.net_order ? a.net_order[t] : t;
    const int p0 = a.net_ptr[n], p1 = a.net_ptr[n + 1];
    Box bx, by;
    bx.init();
    by.init();
    double zhi = -P3D_INF, zlo = P3D_INF;
    for (int k = p0; k < p1; ++k) {  // pass 1: boxes
      double x, y, z;
      int top;
      pins.get(k, x, y, z, top);
      bx.add(x, top);
      by.add(y, top);
      zhi = fmax(zhi, z);
      zlo = fmin(zlo, z);
    }
    const double ex_x = bx.bistratal(), ex_y = by.bistratal();
    const bool split_x = (bx.span(1) + bx.span(0)) > bx.full();  // ties -> full box
    const bool split_y = (by.span(1) + by.span(0)) > by.full();
    acc[3] += ex_x;
    acc[4] += ex_y;
    acc[5] += (bx.cnt[0] > 0 && bx.cnt[1] > 0) ? 1.0 : 0.0;
    const bool dup = a.net_dup && a.net_dup[n];

    WaSum sx[2], sy[2], sz;
    if (PLANAR || CUT) {
      sx[0].init(); sx[1].init(); sy[0].init(); sy[1].init(); sz.init();
      const double fxh = bx.fmaxv(), fxl = bx.fminv(), fyh = by.fmaxv(), fyl = by.fminv();
      for (int k = p0; k < p1; ++k) {  // pass 2: WA sums of the chosen branch
        double x, y, z;
        int top;
        pins.get(k, x, y, z, top);
        if (PLANAR) {
          if (split_x) sx[top].add(x, bx.hi1[top], bx.lo1[top], inv_g); else sx[0].add(x, fxh, fxl, inv_g);
          if (split_y) sy[top].add(y, by.hi1[top], by.lo1[top], inv_g); else sy[0].add(y, fyh, fyl, inv_g);
        }
        if (CUT) sz.add(z, zhi, zlo, inv_g);
      }
      if (PLANAR) {
        acc[0] += split_x ? (sx[0].value() + sx[1].value()) : sx[0].value();
        acc[1] += split_y ? (sy[0].value() + sy[1].value()) : sy[0].value();
      }
      if (CUT) acc[2] += sz.value();
    }
    if (a.want_pins) {
      const double fxh = bx.fmaxv(), fxl = bx.fminv(), fyh = by.fmaxv(), fyl = by.fminv();
      for (int k = p0; k < p1; ++k) {  // pass 3: per-pin outputs
        double x, y, z;
        int top;
        pins.get(k, x, y, z, top);
        double gx = 0.0, gy = 0.0, gc = 0.0, gb = 0.0;
        if (PLANAR) {
          gx = split_x ? sx[top].grad(x, bx.hi1[top], bx.lo1[top], gamma, inv_g)
                       : sx[0].grad(x, fxh, fxl, gamma, inv_g);
          gy = split_y ? sy[top].grad(y, by.hi1[top], by.lo1[top], gamma, inv_g)
                       : sy[0].grad(y, fyh, fyl, gamma, inv_g);
        }
        if (CUT) gc = sz.grad(z, zhi, zlo, gamma, inv_g);
        if (FD) {
          if (!dup) {
            double dw = bx.flip_delta(x, top, ex_x) + by.flip_delta(y, top, ex_y);
            gb = (top ? -dw : dw) * a.scale4;
          } else {
            const int w = a.pin_inst[k];
            bool first = true;
            for (int j = p0; j < k; ++j) if (a.pin_inst[j] == w) { first = false; break; }
            if (first) {
              double up = forced_bistratal(pins, a.pin_inst, p0, p1, w, 1, 0) +
                          forced_bistratal(pins, a.pin_inst, p0, p1, w, 1, 1);
              double dn = forced_bistratal(pins, a.pin_inst, p0, p1, w, 0, 0) +
                          forced_bistratal(pins, a.pin_inst, p0, p1, w, 0, 1);
              gb = a.scale4 * (up - dn);
            }
          }
        }
        const int s = a.pin_slot ? a.pin_slot[k] : k;
        if (a.out4) {
          double4 r;
          r.x = gx; r.y = gy; r.z = gc; r.w = gb;
          reinterpret_cast<double4*>(a.out4)[s] = r;
        } else {
          if (a.gx) a.gx[s] = gx;
          if (a.gy) a.gy[s] = gy;
          if (a.gc) a.gc[s] = gc;
          if (a.gb) a.gb[s] = gb;
        }
      }
    }
  }
  // deterministic grid reduction of the per-net scalars
  if (a.final6 == nullptr) return;
  block_sum<6>(acc, red);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int q = 0; q < 6; ++q) a.partials[q * gridDim.x + blockIdx.x] = acc[q];
  }
  if (last_block(a.counter)) {
    for (int q = 0; q < 6; ++q) {
      double s = ordered_sum(a.partials + q * gridDim.x, gridDim.x, red);
      if (threadIdx.x == 0) a.final6[q] = s;
    }
    if (threadIdx.x == 0 && a.value_out) {
      *a.value_out = a.value_mode == 0 ? a.final6[0] + a.final6[1] : a.final6[2];
    }
  }
}

// ---------------------------------------------------------------------------
// NetBoxes export (per-op API)
// ---------------------------------------------------------------------------
__global__ void netboxes_kernel(NetArgs a, PinsDirect pins, int64_t* cnt, double* min1,
                                double* min2, double* max1, double* max2, double* fmin_,
                                double* fmax_, double* bis) {
  const int n = blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= a.n_net) return;
  Box b;
  b.init();
  for (int k = a.net_ptr[n]; k < a.net_ptr[n + 1]; ++k) {
    double x, y, z;
    int top;
    pins.get(k, x, y, z, top);
    b.add(x, top);
  }
  for (int d = 0; d < 2; ++d) {
    if (cnt) cnt[2 * n + d] = b.cnt[d];
    if (min1) min1[2 * n + d] = b.lo1[d];
    if (min2) min2[2 * n + d] = b.lo2[d];
    if (max1) max1[2 * n + d] = b.hi1[d];
    if (max2) max2[2 * n + d] = b.hi2[d];
  }
  if (fmin_) fmin_[n] = b.fminv();
  if (fmax_) fmax_[n] = b.fmaxv();
  if (bis) bis[n] = b.bistratal();
}

// ---------------------------------------------------------------------------
// owner gather: ordered per-object sums over owner-sorted slots
// (np.bincount(pin_inst, w), gp.py:307-309, wirelength.py:277-279)
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) gather_kernel(GatherArgs a) {
  if (a.halt && *a.halt) return;
  __shared__ double red[32 * 3];
  double acc[3] = {0, 0, 0};
  const double4* in = reinterpret_cast<const double4*>(a.pin4);
  const int stride = gridDim.x * blockDim.x;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < a.n_obj; i += stride) {
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
    for (int s = a.obj_slot_ptr[i]; s < a.obj_slot_ptr[i + 1]; ++s) {
      double4 r = in[s];
      s0 += r.x;
      s1 += r.y;
      s2 += r.z;
      s3 += r.w;
    }
    a.out[i] = s0;
    a.out[a.n_obj + i] = s1;
    a.out[2 * a.n_obj + i] = s2;
    a.out[3 * a.n_obj + i] = s3;
    acc[0] += fabs(s0);
    acc[1] += fabs(s1);
    acc[2] += fabs(s3);
  }
  if (a.final_norms == nullptr) return;
  block_sum<3>(acc, red);
  if (threadIdx.x == 0) {
    for (int q = 0; q < 3; ++q) a.partials[q * gridDim.x + blockIdx.x] = acc[q];
  }
  if (last_block(a.counter)) {
    double nrm[3];
    for (int q = 0; q < 3; ++q) nrm[q] = ordered_sum(a.partials + q * gridDim.x, gridDim.x, red);
    if (threadIdx.x == 0) {
      a.final_norms[0] = nrm[0];
      a.final_norms[1] = nrm[1];
      a.final_norms[2] = nrm[2];
      // Eq. 17 scale (wirelength.py:296-305); 0 encodes the norm-zero branch
      a.final_norms[3] = nrm[2] == 0.0 ? 0.0 : (nrm[0] + nrm[1]) / (2.0 * nrm[2]);
    }
  }
}

// ---------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------
int grid_blocks(int n, int threads, int cap) {
  int b = (n + threads - 1) / threads;
  if (b < 1) b = 1;
  return b < cap ? b : cap;
}

template <class Pins>
static void launch_net(const NetArgs& a, const Pins& pins, bool planar, bool cut, bool fd,
                       cudaStream_t s) {
  const int blocks = a.blocks;
  if (planar && cut && fd) net_kernel<Pins, true, true, true><<<blocks, 256, 0, s>>>(a, pins);
  else if (planar && !cut && !fd) net_kernel<Pins, true, false, false><<<blocks, 256, 0, s>>>(a, pins);
  else if (!planar && cut && !fd) net_kernel<Pins, false, true, false><<<blocks, 256, 0, s>>>(a, pins);
  else if (!planar && !cut && fd) net_kernel<Pins, false, false, true><<<blocks, 256, 0, s>>>(a, pins);
  else net_kernel<Pins, true, true, true><<<blocks, 256, 0, s>>>(a, pins);
}

void launch_net_pos(const NetArgs& a, const double* x, const double* y, const double* z,
                    const double* off, double dz, cudaStream_t s) {
  PinsFromPos p;
  p.x = x; p.y = y; p.z = z;
  p.off = reinterpret_cast<const double4*>(off);
  p.pin_inst = a.pin_inst;
  p.dz2 = dz / 2;
  launch_net(a, p, true, true, true, s);
}

void launch_net_direct(const NetArgs& a, const double* px, const double* py, const double* pz,
                       const uint8_t* top, bool planar, bool cut, bool fd, cudaStream_t s) {
  PinsDirect p;
  p.px = px; p.py = py; p.pz = pz; p.top = top;
  launch_net(a, p, planar, cut, fd, s);
}

void launch_netboxes(const NetArgs& a, const double* c, const uint8_t* top, int64_t* cnt,
                     double* min1, double* min2, double* max1, double* max2, double* fmn,
                     double* fmx, double* bis, cudaStream_t s) {
  PinsDirect p;
  p.px = c; p.py = nullptr; p.pz = nullptr; p.top = top;
  int blocks = (a.n_net + 255) / 256;
  if (blocks < 1) blocks = 1;
  netboxes_kernel<<<blocks, 256, 0, s>>>(a, p, cnt, min1, min2, max1, max2, fmn, fmx, bis);
}

void launch_gather(const GatherArgs& a, cudaStream_t s) {
  gather_kernel<<<a.blocks, 256, 0, s>>>(a);
}

}  // namespace p3d
