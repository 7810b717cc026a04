// K1 (fused-loop variant) — the same math as p3d_wl.cu's net_kernel, laid out
// for bandwidth:
//   * nets are processed grouped by degree; for degree D <= 8 the pins of a
//     bucket are stored transposed ([k][net]) so every pin load of a warp is
//     one coalesced transaction, and the whole net lives in registers
//     (template on D: no local memory, no divergence inside a bucket);
//   * instance centres are gathered from an AoS double4 copy (one 32-byte
//     sector per pin, L2-resident) written by the optimiser step;
//   * pin offsets are float4 (integers / half-integers are exact in fp32);
//   * extrema, spans, crossings and the finite-difference depth term stay in
//     float64 (bit-exact); the weighted-average exponential sums run either in
//     float64 with numpy's operation order (WA_F64) or in float32 on
//     anchor-relative differences (WA_F32: value = (max-min) + fp32 residual;
//     the SURVEY Appendix-B precision plan, within 3e-7 of the fp64
//     trajectory).
// Per-pin outputs: gx, gy, g_cut (float32 or float64) and the FD term (float64)
// at the pin's owner-sorted slot; per-net scalars reduced deterministically.
#include "p3d_common.cuh"
#include "p3d_internal.cuh"

namespace p3d {

namespace {

struct Side {  // extrema of one (net, die) segment on one axis (float64, exact)
  int cnt;
  double hi1, hi2, lo1, lo2;
  __device__ __forceinline__ void init() {
    cnt = 0;
    hi1 = hi2 = -P3D_INF;
    lo1 = lo2 = P3D_INF;
  }
  // top-2 with multiplicity (NetBoxes order statistics, wirelength.py:113-131)
  __device__ __forceinline__ void add(double c) {
    cnt += 1;
    if (c > hi1) { hi2 = hi1; hi1 = c; } else if (c > hi2) { hi2 = c; }
    if (c < lo1) { lo2 = lo1; lo1 = c; } else if (c < lo2) { lo2 = c; }
  }
  __device__ __forceinline__ double span() const { return cnt > 0 ? hi1 - lo1 : 0.0; }
};

// wirelength.py:227-248 for a pin of segment `same` flipping into `other`
__device__ __forceinline__ double flip_delta(const Side& same, const Side& other, double c,
                                             double full, double cur) {
  double sp = 0.0;
  if (same.cnt > 1) sp = ((c == same.hi1) ? same.hi2 : same.hi1) - ((c == same.lo1) ? same.lo2 : same.lo1);
  const double op = fmax(other.hi1, c) - fmin(other.lo1, c);
  return fmax(full, sp + op) - cur;
}

struct Box2 {  // one axis, die 0 (bottom) and die 1 (top)
  Side b, t;
  __device__ __forceinline__ void init() { b.init(); t.init(); }
  __device__ __forceinline__ void add(double c, int d) { if (d) t.add(c); else b.add(c); }
  __device__ __forceinline__ double fmx() const { return fmax(b.hi1, t.hi1); }
  __device__ __forceinline__ double fmn() const { return fmin(b.lo1, t.lo1); }
  __device__ __forceinline__ double full() const { return (b.cnt + t.cnt) > 0 ? fmx() - fmn() : 0.0; }
  __device__ __forceinline__ double flip(double c, int d, double cur) const {
    const double f = full();
    return d ? flip_delta(t, b, c, f, cur) : flip_delta(b, t, c, f, cur);
  }
};

// ---- weighted-average segment sums -------------------------------------------
// float64, numpy operation order (wirelength.py:85-96)
struct Wa64 {
  double s1p, sxp, s1m, sxm;
  __device__ __forceinline__ void init() { s1p = sxp = s1m = sxm = 0.0; }
  __device__ __forceinline__ void add(double v, double hi, double lo, double g, double& ep,
                                      double& em) {
    ep = exp((v - hi) / g);
    em = exp((lo - v) / g);
    s1p += ep;
    sxp += v * ep;
    s1m += em;
    sxm += v * em;
  }
  __device__ __forceinline__ double value(double, double) const {
    return s1p > 0 ? sxp / s1p - sxm / s1m : 0.0;
  }
  __device__ __forceinline__ double grad(double v, double, double, double g, double ep,
                                         double em) const {
    const double vp = sxp / s1p, vm = sxm / s1m;
    return ep / s1p * (1.0 + (v - vp) / g) - em / s1m * (1.0 - (v - vm) / g);
  }
};

// float32 on anchor-relative differences: vp = hi + sum(dp ep)/sum(ep), etc.
struct Wa32 {
  float s1p, sdp, s1m, sdm;
  __device__ __forceinline__ void init() { s1p = sdp = s1m = sdm = 0.f; }
  __device__ __forceinline__ void add(double v, double hi, double lo, float ig, float& ep,
                                      float& em) {
    const float dp = (float)(v - hi), dm = (float)(v - lo);
    ep = __expf(dp * ig);
    em = __expf(-dm * ig);
    s1p += ep;
    sdp += dp * ep;
    s1m += em;
    sdm += dm * em;
  }
  __device__ __forceinline__ double value(double hi, double lo) const {
    if (!(s1p > 0.f)) return 0.0;
    return (hi - lo) + (double)(sdp / s1p - sdm / s1m);
  }
  __device__ __forceinline__ float grad(double v, double hi, double lo, float ig, float ep,
                                        float em) const {
    const float dp = (float)(v - hi), dm = (float)(v - lo);
    const float rp = 1.f / s1p, rm = 1.f / s1m;
    return ep * rp * (1.f + (dp - sdp * rp) * ig) - em * rm * (1.f - (dm - sdm * rm) * ig);
  }
};

template <bool F32>
struct WaSel;
template <>
struct WaSel<false> {
  using W = Wa64;
  using R = double;
  using G = double;
};
template <>
struct WaSel<true> {
  using W = Wa32;
  using R = float;
  using G = float;
};

__device__ __forceinline__ void load_pin(const FusedNetArgs& a, int idx, double& px, double& py,
                                         double& pz, int& top) {
  const int i = a.pin_inst[idx];
  const double4 p = a.pos4[i];
  const float4 o = a.off[idx];
  top = (p.z - a.dz2) > 0.0;
  px = p.x + (double)(top ? o.x : o.z);
  py = p.y + (double)(top ? o.y : o.w);
  pz = p.z;
}

// exact bistratal extent of one axis with every pin of owner w forced to die `forced`
__device__ __noinline__ double forced_ext(const FusedNetArgs& a, int base, int deg, int stride, int w,
                             int forced, int axis) {
  double thi = -P3D_INF, tlo = P3D_INF, bhi = -P3D_INF, blo = P3D_INF, fhi = -P3D_INF,
         flo = P3D_INF;
  int nt = 0, nb = 0;
  for (int k = 0; k < deg; ++k) {
    double x, y, z;
    int t;
    load_pin(a, base + k * stride, x, y, z, t);
    const double c = axis == 0 ? x : y;
    if (a.pin_inst[base + k * stride] == w) t = forced;
    fhi = fmax(fhi, c);
    flo = fmin(flo, c);
    if (t) { nt++; thi = fmax(thi, c); tlo = fmin(tlo, c); } else { nb++; bhi = fmax(bhi, c); blo = fmin(blo, c); }
  }
  const double full = deg > 0 ? fhi - flo : 0.0;
  return fmax(full, (nt ? thi - tlo : 0.0) + (nb ? bhi - blo : 0.0));
}

__device__ __forceinline__ void store_pin(const FusedNetArgs& a, int idx, double gx, double gy,
                                          double gc, double gb) {
  const int s = a.slot[idx];
  a.out_f[s] = make_float4((float)gx, (float)gy, (float)gc, 0.f);
  a.out_fd[s] = gb;
  if (a.out_d) reinterpret_cast<double4*>(a.out_d)[s] = make_double4(gx, gy, gc, gb);
}

// Dup-owner exact path (wirelength.py:280-292): value for the first pin of
// each owner, 0 for its other pins.
__device__ __noinline__ double dup_fd(const FusedNetArgs& a, int base, int deg, int stride,
                                         int k) {
  const int w = a.pin_inst[base + k * stride];
  for (int j = 0; j < k; ++j)
    if (a.pin_inst[base + j * stride] == w) return 0.0;
  const double up = forced_ext(a, base, deg, stride, w, 1, 0) + forced_ext(a, base, deg, stride, w, 1, 1);
  const double dn = forced_ext(a, base, deg, stride, w, 0, 0) + forced_ext(a, base, deg, stride, w, 0, 1);
  return a.scale4 * (up - dn);
}

// One planar axis of a register-resident net: boxes, branch, WA sums of the
// chosen branch, per-pin gradients, FD extent deltas (accumulated into dw).
template <int D, bool F32>
__device__ __forceinline__ void axis_phase(const double (&c)[D], int topm, typename WaSel<F32>::R ig,
                                           double& val, double& exact, bool& crossing,
                                           typename WaSel<F32>::R (&g)[D], double (&dw)[D]) {
  using W = typename WaSel<F32>::W;
  using R = typename WaSel<F32>::R;
  Box2 bx;
  bx.init();
#pragma unroll
  for (int k = 0; k < D; ++k) bx.add(c[k], (topm >> k) & 1);
  const double full = bx.full(), part = bx.t.span() + bx.b.span();
  const double ex = fmax(full, part);
  const bool split = part > full;  // ties resolve to the full box (wirelength.py:186)
  exact = ex;
  crossing = bx.b.cnt > 0 && bx.t.cnt > 0;
  const double fh = bx.fmx(), fl = bx.fmn();
  W w0, w1;
  w0.init();
  w1.init();
#pragma unroll
  for (int k = 0; k < D; ++k) {
    R ep, em;
    const int tp = (topm >> k) & 1;
    if (!split) w0.add(c[k], fh, fl, ig, ep, em);
    else if (tp) w1.add(c[k], bx.t.hi1, bx.t.lo1, ig, ep, em);
    else w0.add(c[k], bx.b.hi1, bx.b.lo1, ig, ep, em);
  }
  val = split ? (w0.value(bx.b.hi1, bx.b.lo1) + w1.value(bx.t.hi1, bx.t.lo1)) : w0.value(fh, fl);
#pragma unroll
  for (int k = 0; k < D; ++k) {
    const int tp = (topm >> k) & 1;
    R ep, em;
    W tmp;
    tmp.init();
    if (!split) {
      tmp.add(c[k], fh, fl, ig, ep, em);
      g[k] = w0.grad(c[k], fh, fl, ig, ep, em);
    } else if (tp) {
      tmp.add(c[k], bx.t.hi1, bx.t.lo1, ig, ep, em);
      g[k] = w1.grad(c[k], bx.t.hi1, bx.t.lo1, ig, ep, em);
    } else {
      tmp.add(c[k], bx.b.hi1, bx.b.lo1, ig, ep, em);
      g[k] = w0.grad(c[k], bx.b.hi1, bx.b.lo1, ig, ep, em);
    }
    dw[k] += bx.flip(c[k], tp, ex);
  }
}

// Register-resident net of compile-time degree D (axis by axis).
template <int D, bool F32>
__device__ __forceinline__ void process_net(const FusedNetArgs& a, int t, double (&acc)[6]) {
  using W = typename WaSel<F32>::W;
  using R = typename WaSel<F32>::R;
  const int base = a.net_base[t];
  const int stride = a.net_stride[t];
  double px[D], py[D], pz[D], dw[D];
  R gx[D], gy[D];
  int topm = 0;
  double zhi = -P3D_INF, zlo = P3D_INF;
#pragma unroll
  for (int k = 0; k < D; ++k) {
    int tp;
    load_pin(a, base + k * stride, px[k], py[k], pz[k], tp);
    topm |= tp << k;
    zhi = fmax(zhi, pz[k]);
    zlo = fmin(zlo, pz[k]);
    dw[k] = 0.0;
  }
  const R ig = F32 ? (R)(1.0 / a.gamma) : (R)a.gamma;  // f32: multiply; f64: divide like numpy
  double v, ex;
  bool cross;
  axis_phase<D, F32>(px, topm, ig, v, ex, cross, gx, dw);
  acc[0] += v;
  acc[3] += ex;
  acc[5] += cross ? 1.0 : 0.0;
  axis_phase<D, F32>(py, topm, ig, v, ex, cross, gy, dw);
  acc[1] += v;
  acc[4] += ex;
  W wz;
  wz.init();
#pragma unroll
  for (int k = 0; k < D; ++k) {
    R ep, em;
    wz.add(pz[k], zhi, zlo, ig, ep, em);
  }
  acc[2] += wz.value(zhi, zlo);
  const bool dup = a.net_dup[t] != 0;
#pragma unroll
  for (int k = 0; k < D; ++k) {
    R ep, em;
    W tmp;
    tmp.init();
    tmp.add(pz[k], zhi, zlo, ig, ep, em);
    const double gc = (double)wz.grad(pz[k], zhi, zlo, ig, ep, em);
    const int tp = (topm >> k) & 1;
    const double gb = dup ? dup_fd(a, base, D, stride, k) : (tp ? -dw[k] : dw[k]) * a.scale4;
    store_pin(a, base + k * stride, gx[k], gy[k], gc, gb);
  }
}

// Any degree: three passes re-loading the pins (large nets; rare).
template <bool F32>
__device__ __noinline__ void process_net_generic(const FusedNetArgs& a, int t, double (&acc)[6]) {
  using W = typename WaSel<F32>::W;
  using R = typename WaSel<F32>::R;
  const int base = a.net_base[t], deg = a.net_deg[t], stride = a.net_stride[t];
  Box2 bx, by;
  bx.init();
  by.init();
  double zhi = -P3D_INF, zlo = P3D_INF;
  for (int k = 0; k < deg; ++k) {
    double x, y, z;
    int tp;
    load_pin(a, base + k * stride, x, y, z, tp);
    bx.add(x, tp);
    by.add(y, tp);
    zhi = fmax(zhi, z);
    zlo = fmin(zlo, z);
  }
  const double ex = fmax(bx.full(), bx.t.span() + bx.b.span());
  const double ey = fmax(by.full(), by.t.span() + by.b.span());
  const bool sx = (bx.t.span() + bx.b.span()) > bx.full();
  const bool sy = (by.t.span() + by.b.span()) > by.full();
  acc[3] += ex;
  acc[4] += ey;
  acc[5] += (bx.b.cnt > 0 && bx.t.cnt > 0) ? 1.0 : 0.0;
  const double fxh = bx.fmx(), fxl = bx.fmn(), fyh = by.fmx(), fyl = by.fmn();
  const R ig = F32 ? (R)(1.0 / a.gamma) : (R)a.gamma;
  W wx0, wx1, wy0, wy1, wz;
  wx0.init(); wx1.init(); wy0.init(); wy1.init(); wz.init();
  for (int k = 0; k < deg; ++k) {
    double x, y, z;
    int tp;
    load_pin(a, base + k * stride, x, y, z, tp);
    R e0, e1;
    if (!sx) wx0.add(x, fxh, fxl, ig, e0, e1);
    else if (tp) wx1.add(x, bx.t.hi1, bx.t.lo1, ig, e0, e1);
    else wx0.add(x, bx.b.hi1, bx.b.lo1, ig, e0, e1);
    if (!sy) wy0.add(y, fyh, fyl, ig, e0, e1);
    else if (tp) wy1.add(y, by.t.hi1, by.t.lo1, ig, e0, e1);
    else wy0.add(y, by.b.hi1, by.b.lo1, ig, e0, e1);
    wz.add(z, zhi, zlo, ig, e0, e1);
  }
  acc[0] += sx ? (wx0.value(bx.b.hi1, bx.b.lo1) + wx1.value(bx.t.hi1, bx.t.lo1)) : wx0.value(fxh, fxl);
  acc[1] += sy ? (wy0.value(by.b.hi1, by.b.lo1) + wy1.value(by.t.hi1, by.t.lo1)) : wy0.value(fyh, fyl);
  acc[2] += wz.value(zhi, zlo);
  const bool dup = a.net_dup[t] != 0;
  for (int k = 0; k < deg; ++k) {
    double x, y, z;
    int tp;
    load_pin(a, base + k * stride, x, y, z, tp);
    R e0, e1;
    W d;
    d.init();
    double gx, gy;
    if (!sx) { d.add(x, fxh, fxl, ig, e0, e1); gx = (double)wx0.grad(x, fxh, fxl, ig, e0, e1); }
    else if (tp) { d.add(x, bx.t.hi1, bx.t.lo1, ig, e0, e1); gx = (double)wx1.grad(x, bx.t.hi1, bx.t.lo1, ig, e0, e1); }
    else { d.add(x, bx.b.hi1, bx.b.lo1, ig, e0, e1); gx = (double)wx0.grad(x, bx.b.hi1, bx.b.lo1, ig, e0, e1); }
    if (!sy) { d.add(y, fyh, fyl, ig, e0, e1); gy = (double)wy0.grad(y, fyh, fyl, ig, e0, e1); }
    else if (tp) { d.add(y, by.t.hi1, by.t.lo1, ig, e0, e1); gy = (double)wy1.grad(y, by.t.hi1, by.t.lo1, ig, e0, e1); }
    else { d.add(y, by.b.hi1, by.b.lo1, ig, e0, e1); gy = (double)wy0.grad(y, by.b.hi1, by.b.lo1, ig, e0, e1); }
    d.add(z, zhi, zlo, ig, e0, e1);
    const double gc = (double)wz.grad(z, zhi, zlo, ig, e0, e1);
    double gb;
    if (!dup) {
      const double dwv = bx.flip(x, tp, ex) + by.flip(y, tp, ey);
      gb = (tp ? -dwv : dwv) * a.scale4;
    } else {
      gb = dup_fd(a, base, deg, stride, k);
    }
    store_pin(a, base + k * stride, gx, gy, gc, gb);
  }
}

template <bool F32>
__global__ void __launch_bounds__(256, F32 ? 2 : 1) fused_net_kernel(FusedNetArgs a) {
  if (a.halt && *a.halt) return;
  __shared__ double red[32 * 6];
  if (a.gamma_ptr) a.gamma = *a.gamma_ptr;
  double acc[6] = {0, 0, 0, 0, 0, 0};
  const int stride = gridDim.x * blockDim.x;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < a.n_net; t += stride) {
    switch (a.net_deg[t]) {
      case 2: process_net<2, F32>(a, t, acc); break;
      case 3: process_net<3, F32>(a, t, acc); break;
      case 4: process_net<4, F32>(a, t, acc); break;
      case 5: process_net<5, F32>(a, t, acc); break;
      case 6: process_net<6, F32>(a, t, acc); break;
      default: process_net_generic<F32>(a, t, acc); break;
    }
  }
  block_sum<6>(acc, red);
  if (threadIdx.x == 0)
    for (int q = 0; q < 6; ++q) a.partials[q * gridDim.x + blockIdx.x] = acc[q];
  if (last_block(a.counter)) {
    for (int q = 0; q < 6; ++q) {
      const double s = ordered_sum(a.partials + q * gridDim.x, gridDim.x, red);
      if (threadIdx.x == 0) a.final6[q] = s;
    }
  }
}

// owner gather of the split outputs: per object, ordered fp64 sums over slots
__global__ void __launch_bounds__(256) fused_gather_kernel(FusedGatherArgs a) {
  if (a.halt && *a.halt) return;
  __shared__ double red[32 * 3];
  double acc[3] = {0, 0, 0};
  const int stride = gridDim.x * blockDim.x;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < a.n_obj; i += stride) {
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
    const int b = a.obj_slot_ptr[i], e = a.obj_slot_ptr[i + 1];
    if (a.in_d) {
      const double4* in = reinterpret_cast<const double4*>(a.in_d);
      for (int s = b; s < e; ++s) {
        const double4 r = in[s];
        s0 += r.x; s1 += r.y; s2 += r.z; s3 += r.w;
      }
    } else {
      for (int s = b; s < e; ++s) {
        const float4 r = a.in_f[s];
        s0 += (double)r.x; s1 += (double)r.y; s2 += (double)r.z;
        s3 += a.in_fd[s];
      }
    }
    a.out[i] = s0;
    a.out[a.n_obj + i] = s1;
    a.out[2 * a.n_obj + i] = s2;
    a.out[3 * a.n_obj + i] = s3;
    acc[0] += fabs(s0);
    acc[1] += fabs(s1);
    acc[2] += fabs(s3);
  }
  block_sum<3>(acc, red);
  if (threadIdx.x == 0)
    for (int q = 0; q < 3; ++q) a.partials[q * gridDim.x + blockIdx.x] = acc[q];
  if (last_block(a.counter)) {
    double n[3];
    for (int q = 0; q < 3; ++q) n[q] = ordered_sum(a.partials + q * gridDim.x, gridDim.x, red);
    if (threadIdx.x == 0) {
      a.final_norms[0] = n[0];
      a.final_norms[1] = n[1];
      a.final_norms[2] = n[2];
      a.final_norms[3] = n[2] == 0.0 ? 0.0 : (n[0] + n[1]) / (2.0 * n[2]);  // Eq. 17
    }
  }
}

}  // namespace

void launch_fused_net(const FusedNetArgs& a, bool f32, cudaStream_t s) {
  if (f32) fused_net_kernel<true><<<a.blocks, 256, 0, s>>>(a);
  else fused_net_kernel<false><<<a.blocks, 256, 0, s>>>(a);
}

void launch_fused_gather(const FusedGatherArgs& a, cudaStream_t s) {
  fused_gather_kernel<<<a.blocks, 256, 0, s>>>(a);
}

}  // namespace p3d
