// K1 (fused-loop variant) — the same math as p3d_wl.cu's net_kernel, laid out
// for bandwidth and latency:
//   * nets are grouped by degree; each degree bucket stores its pins
//     transposed ([pin k][net j]) so a warp that owns 32 nets of one bucket
//     loads pin k of all 32 nets in one coalesced transaction;
//   * a warp first STAGES its 32*D pins (owner gather from the AoS double4
//     copy of the instance centres — one 32-byte sector per pin, L2-resident —
//     plus float4 offsets) into per-lane shared-memory columns, with all D
//     gathers of a lane independent (memory-level parallelism), then each lane
//     evaluates its own net from shared memory (no register spills, no local
//     memory);
//   * per-pin results (gx, gy, g_cut, FD term) are written as one record per
//     pin in the same coalesced order; the owner gather reads them through an
//     owner-sorted index list (deterministic per-object sums);
//   * extrema, spans, crossings and the finite-difference depth term are
//     float64 and bit-exact; the weighted-average exponential sums run in
//     float64 with numpy's operation order (default) or, opt-in, float32 on
//     anchor-relative differences (SURVEY App. B plan).
// Nets with degree outside [2, kMaxStagedDeg] take a per-thread generic path.
#include <algorithm>

#include "p3d_common.cuh"
#include "p3d_internal.cuh"

namespace p3d {

namespace {

#ifndef P3D_BOX_SELECT
#define P3D_BOX_SELECT 1
#endif

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
    push(c, c);
  }
  // the same update without branches: hi2' = max(hi2, min(hi1, h)) and
  // hi1' = max(hi1, h) pick exactly the values of the if/else chain; h = -inf
  // (l = +inf) leaves the side unchanged
  __device__ __forceinline__ void push(double h, double l) {
#if P3D_BOX_SELECT
    hi2 = dmax(hi2, dmin(hi1, h));
    hi1 = dmax(hi1, h);
    lo2 = dmin(lo2, dmax(lo1, l));
    lo1 = dmin(lo1, l);
#else
    if (h > hi1) { hi2 = hi1; hi1 = h; } else if (h > hi2) { hi2 = h; }
    if (l < lo1) { lo2 = lo1; lo1 = l; } else if (l < lo2) { lo2 = l; }
#endif
  }
  __device__ __forceinline__ double span() const { return cnt > 0 ? hi1 - lo1 : 0.0; }
};

// wirelength.py:227-248 for a pin of segment `same` flipping into `other`
__device__ __forceinline__ double flip_delta(const Side& same, const Side& other, double c,
                                             double full, double cur) {
  double sp = 0.0;
  if (same.cnt > 1) sp = ((c == same.hi1) ? same.hi2 : same.hi1) - ((c == same.lo1) ? same.lo2 : same.lo1);
  const double op = dmax(other.hi1, c) - dmin(other.lo1, c);
  return dmax(full, sp + op) - cur;
}

struct Box2 {  // one axis, die 0 (bottom) and die 1 (top)
  Side b, t;
  __device__ __forceinline__ void init() { b.init(); t.init(); }
  __device__ __forceinline__ void add(double c, int d) {
#if P3D_BOX_SELECT
    t.push(d ? c : -P3D_INF, d ? c : P3D_INF);
    b.push(d ? -P3D_INF : c, d ? P3D_INF : c);
    t.cnt += d;
    b.cnt += 1 - d;
#else
    if (d) t.add(c); else b.add(c);
#endif
  }
  __device__ __forceinline__ double fmx() const { return dmax(b.hi1, t.hi1); }
  __device__ __forceinline__ double fmn() const { return dmin(b.lo1, t.lo1); }
  __device__ __forceinline__ double full() const { return (b.cnt + t.cnt) > 0 ? fmx() - fmn() : 0.0; }
  // wirelength.py:227-248 with the pin's own segment / the other segment picked by selects
  __device__ __forceinline__ double flip(double c, int d, double full_, double cur) const {
    const int scnt = d ? t.cnt : b.cnt;
    const double shi1 = d ? t.hi1 : b.hi1, shi2 = d ? t.hi2 : b.hi2;
    const double slo1 = d ? t.lo1 : b.lo1, slo2 = d ? t.lo2 : b.lo2;
    const double ohi1 = d ? b.hi1 : t.hi1, olo1 = d ? b.lo1 : t.lo1;
    const double sp = scnt > 1 ? ((c == shi1) ? shi2 : shi1) - ((c == slo1) ? slo2 : slo1) : 0.0;
    const double op = dmax(ohi1, c) - dmin(olo1, c);
    return dmax(full_, sp + op) - cur;
  }
};

// ---- weighted-average segment sums -------------------------------------------
// exp(x) for x <= 0 (every WA argument is (v - max)/gamma or (min - v)/gamma).
// Default: the table-free polynomial below (P3D_EXP_POLY, measured faster: the
// table load was the kernel's top stall; re-measured late in round 2 with the
// table in L1 or in shared memory: K1 +7 / +5.5 us, -2.3% / -1.7% it/s).  Alternative (-DP3D_EXP_POLY=0):
// x = (64 m + k) ln2/64 + r with |r| <= ln2/128: exp(x) = 2^m T[k] (1 + q(r)),
// T[k] = 2^(k/64) (64-entry table), q a degree-6 Taylor polynomial evaluated
// with short dependency chains (Estrin) — this kernel is latency-bound at the
// occupancy its shared-memory columns allow.  <= 2 ulp against numpy's exp
// over [-708, 0]; results below 2^-1022 flush to 0 (each segment sum holds its
// anchor pin's exp(0) = 1, so this is invisible).
__device__ const double kExp2Tab[64] = {
    1.0, 1.0108892860517005, 1.0218971486541166, 1.0330248790212284,
    1.0442737824274138, 1.0556451783605572, 1.0671404006768237, 1.0787607977571199,
    1.0905077326652577, 1.102382583307841, 1.1143867425958924, 1.1265216186082418,
    1.1387886347566916, 1.1511892299529827, 1.1637248587775775, 1.1763969916502812,
    1.189207115002721, 1.202156731452703, 1.215247359980469, 1.22848053610687,
    1.241857812073484, 1.255380757024691, 1.2690509571917332, 1.2828700160787783,
    1.2968395546510096, 1.3109612115247644, 1.3252366431597413, 1.339667524053303,
    1.3542555469368927, 1.3690024229745905, 1.383909881963832, 1.3989796725383112,
    1.4142135623730951, 1.42961333839197, 1.4451808069770467, 1.460917794180647,
    1.4768261459394993, 1.4929077282912648, 1.5091644275934228, 1.5255981507445384,
    1.5422108254079407, 1.559004400237837, 1.5759808451078865, 1.593142151342267,
    1.6104903319492543, 1.6280274218573478, 1.645755478153965, 1.6636765803267364,
    1.681792830507429, 1.7001063537185235, 1.718619298122478, 1.7373338352737062,
    1.7562521603732995, 1.7753764925265212, 1.7947090750031072, 1.8142521755003989,
    1.8340080864093424, 1.8539791250833855, 1.8741676341103, 1.8945759815869656,
    1.9152065613971474, 1.9360617934922943, 1.9571441241754002, 1.978456026387951};

#ifndef P3D_EXP_POLY
#define P3D_EXP_POLY 1
#endif
#ifndef P3D_EXP_CONST
#define P3D_EXP_CONST 1
#endif
#ifndef P3D_K1_EARLY
#define P3D_K1_EARLY 1
#endif
#if P3D_EXP_POLY
// Table-free variant: n = rint(x / ln 2), Cody-Waite r (|r| <= ln2/2), degree-13
// Taylor polynomial by Horner (<= 1.2 ulp over [-708, 0]); no memory access.
// The coefficients live in constant memory so every DFMA takes its constant
// as a c[][] operand: as immediates the compiler rematerialised each fp64
// constant with two UMOVs per use (9% of K1's instructions).
__constant__ double kExpPoly[17] = {
    1.4426950408889634074,     // 1 / ln 2
    0.693147180369123816490,   // ln 2 (high part)
    1.9082149292705877e-10,    // ln 2 (low part)
    1.6059043836821613e-10,    // 1/13!
    2.08767569878680989792e-09,  // 1/12!
    2.50521083854417187751e-08,  // 1/11!
    2.75573192239858906526e-07,  // 1/10!
    2.75573192239858906526e-06,  // 1/9!
    2.48015873015873015873e-05,  // 1/8!
    1.98412698412698412698e-04,  // 1/7!
    1.38888888888888888889e-03,  // 1/6!
    8.33333333333333333333e-03,  // 1/5!
    4.16666666666666666667e-02,  // 1/4!
    1.66666666666666666667e-01,  // 1/3!
    0.5, 1.0, 1.0};
__device__ __forceinline__ double exp_neg(double x) {
#ifdef P3D_PROBE_EXP  // timing probe only: a 2-FMA stand-in (results wrong)
  return fma(x, fma(x, 0.5, 1.0), 1.0);
#endif
#if P3D_EXP_CONST
  const double* c = kExpPoly;
#else
  constexpr double c[17] = {1.4426950408889634074, 0.693147180369123816490,
                            1.9082149292705877e-10, 1.6059043836821613e-10,
                            2.08767569878680989792e-09, 2.50521083854417187751e-08,
                            2.75573192239858906526e-07, 2.75573192239858906526e-06,
                            2.48015873015873015873e-05, 1.98412698412698412698e-04,
                            1.38888888888888888889e-03, 8.33333333333333333333e-03,
                            4.16666666666666666667e-02, 1.66666666666666666667e-01,
                            0.5, 1.0, 1.0};
#endif
  const double n = rint(x * c[0]);
  const double r = fma(-n, c[2], fma(-n, c[1], x));
  double p = c[3];
#pragma unroll
  for (int k = 4; k < 17; ++k) p = fma(p, r, c[k]);
  const double sc = __longlong_as_double((long long)((int)n + 1023) << 52);
  return x < -708.0 ? 0.0 : p * sc;
}
#else
__device__ __forceinline__ double exp_neg(double x) {
  const double n = rint(x * 92.332482616893656877);  // 64 / ln 2
  const double r = fma(-n, 2.572804622327669e-14, fma(-n, 0.010830424696223417, x));
  const int ni = (int)n;
  const double r2 = r * r;
  const double a = fma(r, 1.6666666666666666e-01, 0.5);            // 1/2 + r/6
  const double b = fma(r, 8.333333333333333e-03, 4.1666666666666664e-02);  // 1/24 + r/120
  const double c = fma(r2, 1.3888888888888889e-03, b);             // + r^2/720
  const double q = fma(r2, fma(r2, c, a), r);                      // r + r^2 a + r^4 c
  const double t = __ldg(&kExp2Tab[ni & 63]);
  const double sc = __longlong_as_double((long long)((ni >> 6) + 1023) << 52);
  return x < -708.0 ? 0.0 : fma(t, q, t) * sc;
}
#endif

// float64 WA sums with numpy's structure (wirelength.py:85-96): value
// sxp/s1p - sxm/s1m, gradient ep/s1p (1 + (v - vp)/g) - em/s1m (1 - (v - vm)/g);
// 1/gamma and the per-segment reciprocals are hoisted (<= 1 ulp differences).
template <class R>
struct GradK {  // per-segment constants of the per-pin WA gradient
  R rp, rm;
  double vp, vm;
  // ep/s1p (1 + (v - vp)/g) - em/s1m (1 - (v - vm)/g)  (wirelength.py:94-96)
  __device__ __forceinline__ R grad(double v, R ig, R ep, R em) const {
    return ep * rp * ((R)1 + (R)(v - vp) * ig) - em * rm * ((R)1 - (R)(v - vm) * ig);
  }
};

struct Wa64 {
  using R = double;
  double s1p, sxp, s1m, sxm, rp, rm, vp, vm;
  __device__ __forceinline__ void init() { s1p = sxp = s1m = sxm = 0.0; }
  __device__ static __forceinline__ void term(double v, double hi, double lo, double ig, double& ep,
                                              double& em) {
    ep = exp_neg((v - hi) * ig);
    em = exp_neg((lo - v) * ig);
  }
  // the ep of the lower of two pins, (lo - hi)/g (the other exponentials of a
  // 2-pin segment are exp(0) = 1 exactly, as term() would return them)
  __device__ static __forceinline__ double gap(double hi, double lo, double ig) {
    return exp_neg((lo - hi) * ig);
  }
  __device__ __forceinline__ void acc(double v, double, double, double ep, double em, double on) {
    s1p = fma(on, ep, s1p);
    sxp = fma(on, v * ep, sxp);
    s1m = fma(on, em, s1m);
    sxm = fma(on, v * em, sxm);
  }
  __device__ __forceinline__ void finalize() {
    rp = s1p > 0 ? 1.0 / s1p : 0.0;
    rm = s1m > 0 ? 1.0 / s1m : 0.0;
    vp = sxp * rp;
    vm = sxm * rm;
  }
  __device__ __forceinline__ double value(double, double) const { return s1p > 0 ? vp - vm : 0.0; }
  __device__ __forceinline__ GradK<double> gk(double, double) const { return {rp, rm, vp, vm}; }
  __device__ __forceinline__ double grad(double v, double, double, double ig, double ep,
                                         double em) const {
    return ep * rp * (1.0 + (v - vp) * ig) - em * rm * (1.0 - (v - vm) * ig);
  }
};

// float32 on anchor-relative differences: vp = hi + sum(dp ep)/sum(ep), etc.
struct Wa32 {
  using R = float;
  float s1p, sdp, s1m, sdm, rp, rm, mp, mm;
  __device__ __forceinline__ void init() { s1p = sdp = s1m = sdm = 0.f; }
  __device__ static __forceinline__ void term(double v, double hi, double lo, float ig, float& ep,
                                              float& em) {
    ep = __expf((float)(v - hi) * ig);
    em = __expf(-(float)(v - lo) * ig);
  }
  __device__ static __forceinline__ float gap(double hi, double lo, float ig) {
    return __expf((float)(lo - hi) * ig);
  }
  __device__ __forceinline__ void acc(double v, double hi, double lo, float ep, float em, float on) {
    const float dp = (float)(v - hi), dm = (float)(v - lo);
    s1p = fmaf(on, ep, s1p);
    sdp = fmaf(on, dp * ep, sdp);
    s1m = fmaf(on, em, s1m);
    sdm = fmaf(on, dm * em, sdm);
  }
  __device__ __forceinline__ void finalize() {
    rp = s1p > 0.f ? 1.f / s1p : 0.f;
    rm = s1m > 0.f ? 1.f / s1m : 0.f;
    mp = sdp * rp;
    mm = sdm * rm;
  }
  __device__ __forceinline__ double value(double hi, double lo) const {
    return s1p > 0.f ? (hi - lo) + (double)(mp - mm) : 0.0;
  }
  __device__ __forceinline__ GradK<float> gk(double hi, double lo) const {
    return {rp, rm, hi + (double)mp, lo + (double)mm};
  }
  __device__ __forceinline__ float grad(double v, double hi, double lo, float ig, float ep,
                                        float em) const {
    const float dp = (float)(v - hi), dm = (float)(v - lo);
    return ep * rp * (1.f + (dp - mp) * ig) - em * rm * (1.f - (dm - mm) * ig);
  }
};

template <bool F32>
struct WaSel;
template <>
struct WaSel<false> {
  using W = Wa64;
  using R = double;
};
template <>
struct WaSel<true> {
  using W = Wa32;
  using R = float;
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
    fhi = dmax(fhi, c);
    flo = dmin(flo, c);
    if (t) { nt++; thi = dmax(thi, c); tlo = dmin(tlo, c); } else { nb++; bhi = dmax(bhi, c); blo = dmin(blo, c); }
  }
  const double full = deg > 0 ? fhi - flo : 0.0;
  return dmax(full, (nt ? thi - tlo : 0.0) + (nb ? bhi - blo : 0.0));
}

// one output record per pin, written at its owner-sorted slot (the owner
// gather then streams each object's records contiguously)
__device__ __forceinline__ void store_pin(const FusedNetArgs& a, int idx, double gx, double gy,
                                          double gc, double gb) {
  const int s = a.slot[idx];
  if (a.out_d) reinterpret_cast<double4*>(a.out_d)[s] = make_double4(gx, gy, gc, gb);
  else a.out_f[s] = make_float4((float)gx, (float)gy, (float)gc, (float)gb);
}


// ---- L2 residency hints: the per-pin records are written here and read back
// by the owner gather right after, so they are stored with an evict-last
// policy; the bucketed pin streams (owner, offsets, slot) are read once per
// iteration and loaded evict-first.  (-DP3D_L2_HINTS=0 disables.)
#ifndef P3D_L2_HINTS
#define P3D_L2_HINTS 1
#endif
__device__ __forceinline__ void store_rec(double* base, int slot, double a, double b, double c,
                                          double d) {
#ifdef P3D_PROBE_NOSTORE  // timing probe only: the record values are kept live, not stored
  asm volatile("" ::"d"(a), "d"(b), "d"(c), "d"(d), "r"(slot));
  return;
#endif
  double* p = base + 4 * (long long)slot;
#if P3D_L2_HINTS
  unsigned long long pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;" ::"l"(p), "d"(a), "d"(b),
               "l"(pol)
               : "memory");
  asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;" ::"l"(p + 2), "d"(c), "d"(d),
               "l"(pol)
               : "memory");
#else
  reinterpret_cast<double4*>(p)[0] = make_double4(a, b, c, d);
#endif
}

template <class T>
__device__ __forceinline__ T ld_stream(const T* p) {
#if P3D_L2_HINTS
  return __ldcs(p);  // streaming: evict-first in L1 and L2
#else
  return *p;
#endif
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

// segment of one pin on one axis: anchors of the chosen WA branch
struct SegSel {
  double hi, lo;
  bool upper;  // true: the die-1 (top) partial segment
};
__device__ __forceinline__ SegSel seg_of(const Box2& bx, bool split, int tp) {
  SegSel s;
  s.upper = split && tp;
  s.hi = split ? (tp ? bx.t.hi1 : bx.b.hi1) : bx.fmx();
  s.lo = split ? (tp ? bx.t.lo1 : bx.b.lo1) : bx.fmn();
  return s;
}

// Any degree: three passes re-loading the pins (large / duplicate-owner nets).
template <bool F32>
__device__ __noinline__ void process_net_generic(const FusedNetArgs& a, int t, double (&acc)[6]) {
  using W = typename WaSel<F32>::W;
  using R = typename WaSel<F32>::R;
  const int base = a.net_base[t], deg = a.net_deg[t], stride = a.net_stride[t];
  const uint8_t nd = a.net_dup[t];
  const double pm = (nd & 2) ? 0.0 : 1.0;  // value counted by another rank (halo mode)
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
    zhi = dmax(zhi, z);
    zlo = dmin(zlo, z);
  }
  const double fx = bx.full(), fy = by.full();
  const double ex = dmax(fx, bx.t.span() + bx.b.span());
  const double ey = dmax(fy, by.t.span() + by.b.span());
  const bool sx = (bx.t.span() + bx.b.span()) > fx;
  const bool sy = (by.t.span() + by.b.span()) > fy;
  acc[3] += pm * ex;
  acc[4] += pm * ey;
  acc[5] += pm * ((bx.b.cnt > 0 && bx.t.cnt > 0) ? 1.0 : 0.0);
  const R ig = (R)a.inv_gamma;
  W wx0, wx1, wy0, wy1, wz;
  wx0.init(); wx1.init(); wy0.init(); wy1.init(); wz.init();
  for (int k = 0; k < deg; ++k) {
    double x, y, z;
    int tp;
    load_pin(a, base + k * stride, x, y, z, tp);
    R ep, em;
    const SegSel gx = seg_of(bx, sx, tp), gy = seg_of(by, sy, tp);
    W::term(x, gx.hi, gx.lo, ig, ep, em);
    wx0.acc(x, gx.hi, gx.lo, ep, em, gx.upper ? 0 : 1);
    wx1.acc(x, gx.hi, gx.lo, ep, em, gx.upper ? 1 : 0);
    W::term(y, gy.hi, gy.lo, ig, ep, em);
    wy0.acc(y, gy.hi, gy.lo, ep, em, gy.upper ? 0 : 1);
    wy1.acc(y, gy.hi, gy.lo, ep, em, gy.upper ? 1 : 0);
    W::term(z, zhi, zlo, ig, ep, em);
    wz.acc(z, zhi, zlo, ep, em, 1);
  }
  wx0.finalize(); wx1.finalize(); wy0.finalize(); wy1.finalize(); wz.finalize();
  acc[0] += pm * (sx ? (wx0.value(bx.b.hi1, bx.b.lo1) + wx1.value(bx.t.hi1, bx.t.lo1)) : wx0.value(bx.fmx(), bx.fmn()));
  acc[1] += pm * (sy ? (wy0.value(by.b.hi1, by.b.lo1) + wy1.value(by.t.hi1, by.t.lo1)) : wy0.value(by.fmx(), by.fmn()));
  acc[2] += pm * wz.value(zhi, zlo);
  const bool dup = (nd & 1) != 0;
  for (int k = 0; k < deg; ++k) {
    double x, y, z;
    int tp;
    load_pin(a, base + k * stride, x, y, z, tp);
    R ep, em;
    const SegSel gx = seg_of(bx, sx, tp), gy = seg_of(by, sy, tp);
    W::term(x, gx.hi, gx.lo, ig, ep, em);
    const double ggx = (double)(gx.upper ? wx1 : wx0).grad(x, gx.hi, gx.lo, ig, ep, em);
    W::term(y, gy.hi, gy.lo, ig, ep, em);
    const double ggy = (double)(gy.upper ? wy1 : wy0).grad(y, gy.hi, gy.lo, ig, ep, em);
    W::term(z, zhi, zlo, ig, ep, em);
    const double gc = (double)wz.grad(z, zhi, zlo, ig, ep, em);
    double gb;
    if (!dup) {
      const double dwv = bx.flip(x, tp, fx, ex) + by.flip(y, tp, fy, ey);
      gb = (tp ? -dwv : dwv) * a.scale4;
    } else {
      gb = dup_fd(a, base, deg, stride, k);
    }
    store_pin(a, base + k * stride, ggx, ggy, gc, gb);
  }
}

// the per-pin loops of the staged path: not unrolled by default (register
// budget); -DP3D_K1_FULL_UNROLL unrolls them (D is a template constant)
#ifdef P3D_K1_FULL_UNROLL
#define P3D_K1_LOOP_UNROLL _Pragma("unroll")
#else
#define P3D_K1_LOOP_UNROLL _Pragma("unroll 1")
#endif
#ifndef P3D_FLIP_SELECT
#define P3D_FLIP_SELECT 1
#endif
#ifndef P3D_K1_TRIPLE
#define P3D_K1_TRIPLE 1
#endif
#ifndef P3D_K1_RTD
#define P3D_K1_RTD 1
#endif
#ifndef P3D_K1_MINB
#define P3D_K1_MINB 4
#endif

constexpr int kMaxStagedDeg = 6;
constexpr int kWarpsPerBlock = 4;

// per-lane shared-memory columns of one warp (index [k][lane])
template <bool F32>
struct WarpCols {
  using R = typename WaSel<F32>::R;
  double px[kMaxStagedDeg][32], py[kMaxStagedDeg][32];
  double pz[kMaxStagedDeg][32];  // z for the cut phase, then reused as the FD accumulator
  double gc[kMaxStagedDeg][32];  // z-cut gradient
  R ep[kMaxStagedDeg][32], em[kMaxStagedDeg][32];
};

// One planar axis of a staged net (degree D, fully unrolled: every shared-
// memory column offset is an immediate): boxes, branch, WA sums of the chosen
// branch, per-pin gradients (written over the consumed coordinate column), FD
// extent deltas (accumulated into pz, which holds the FD accumulator by this
// phase).  Per-pin segment choices are selects of hoisted per-segment
// constants; the FD delta is evaluated for both dies and selected.  The
// second segment is finalised only for split nets.
template <int D, bool F32>
__device__ __forceinline__ void staged_axis(double (&c)[kMaxStagedDeg][32], WarpCols<F32>& sm,
                                            int lane, int topm, typename WaSel<F32>::R ig,
                                            double& val, double& exact, bool& crossing, int nd) {
  using W = typename WaSel<F32>::W;
  using R = typename WaSel<F32>::R;
  const int DD = D ? D : nd;  // D = 0: runtime degree (one code path for every degree)
  Box2 bx;
  bx.init();
#pragma unroll
  for (int k = 0; k < (D ? D : kMaxStagedDeg); ++k)
    if (k < DD) bx.add(c[k][lane], (topm >> k) & 1);
  const double full = bx.full(), part = bx.t.span() + bx.b.span();
  const double ex = dmax(full, part);
  const bool split = part > full;  // ties resolve to the full box (wirelength.py:186)
  exact = ex;
  crossing = bx.b.cnt > 0 && bx.t.cnt > 0;
  // segment 0: the whole net (unsplit) or die 0; segment 1: die 1 (split only)
  const double h0 = split ? bx.b.hi1 : bx.fmx(), l0 = split ? bx.b.lo1 : bx.fmn();
  const double h1 = bx.t.hi1, l1 = bx.t.lo1;
  const int umask = split ? topm : 0;
  W w0, w1;
  w0.init();
  w1.init();
P3D_K1_LOOP_UNROLL
  for (int k = 0; k < DD; ++k) {
    const double v = c[k][lane];
    const bool up = (umask >> k) & 1;
    R ep, em;
    W::term(v, up ? h1 : h0, up ? l1 : l0, ig, ep, em);
    sm.ep[k][lane] = ep;
    sm.em[k][lane] = em;
    w0.acc(v, h0, l0, ep, em, up ? 0 : 1);
    w1.acc(v, h1, l1, ep, em, up ? 1 : 0);
  }
  w0.finalize();
  GradK<R> k1 = {};
  val = w0.value(h0, l0);
  if (split) {
    w1.finalize();
    val += w1.value(h1, l1);
    k1 = w1.gk(h1, l1);
  }
  const GradK<R> k0 = w0.gk(h0, l0);
P3D_K1_LOOP_UNROLL
  for (int k = 0; k < DD; ++k) {
    const double v = c[k][lane];
    const bool up = (umask >> k) & 1;
    const GradK<R> gk = {up ? k1.rp : k0.rp, up ? k1.rm : k0.rm, up ? k1.vp : k0.vp,
                         up ? k1.vm : k0.vm};
#if P3D_FLIP_SELECT  // select the pin's sides first, one flip evaluation
    sm.pz[k][lane] += bx.flip(v, (topm >> k) & 1, full, ex);
#else
    const double fb = flip_delta(bx.b, bx.t, v, full, ex), ft = flip_delta(bx.t, bx.b, v, full, ex);
    sm.pz[k][lane] += ((topm >> k) & 1) ? ft : fb;
#endif
    c[k][lane] = (double)gk.grad(v, ig, sm.ep[k][lane], sm.em[k][lane]);
  }
}

// Stage the 32 nets of degree D owned by one warp (D independent owner gathers
// per lane), then evaluate one net per lane from shared memory.
template <int D, bool F32>
__device__ __forceinline__ bool stage_pins(const FusedNetArgs& a, const int4 tk, int t0,
                                           WarpCols<F32>& sm, int lane, int& topm, double& zhi,
                                           double& zlo, double& pm) {
  const int nb = tk.y, j = tk.z + lane;
  if (j >= nb) return false;
  const uint8_t nd = a.net_dup[t0 + j];
#if !P3D_K1_EARLY
  if (nd & 1) return false;  // duplicate-owner nets: generic kernel
#endif
  pm = (nd & 2) ? 0.0 : 1.0;  // value counted by another rank (halo mode)
  const int pin0 = tk.x + j;
  constexpr int KM = D ? D : kMaxStagedDeg;
  const int DD = D ? D : tk.w;
  int inst[KM];
  float4 off[KM];
#pragma unroll
  for (int k = 0; k < KM; ++k) {
    if (k >= DD) break;
    inst[k] = ld_stream(a.pin_inst + pin0 + k * nb);
    off[k] = ld_stream(a.off + pin0 + k * nb);
  }
#if P3D_K1_EARLY
  if (nd & 1) return false;  // duplicate-owner nets: generic kernel
#endif
  topm = 0;
  zhi = -P3D_INF;
  zlo = P3D_INF;
#pragma unroll
  for (int k = 0; k < KM; ++k) {
    if (k >= DD) break;
#ifdef P3D_PROBE_NOGATHER  // timing probe only: every pin reads one line (results wrong)
    const double4 p = a.pos4[inst[k] & 31];
#else
    const double4 p = a.pos4[inst[k]];
#endif
    const int tp = (p.z - a.dz2) > 0.0;
    topm |= tp << k;
    sm.px[k][lane] = p.x + (double)(tp ? off[k].x : off[k].z);
    sm.py[k][lane] = p.y + (double)(tp ? off[k].y : off[k].w);
    sm.pz[k][lane] = p.z;
    zhi = dmax(zhi, p.z);
    zlo = dmin(zlo, p.z);
  }
  return true;
}

template <int D, bool F32>
__device__ __forceinline__ void staged_eval(const FusedNetArgs& a, int pin0, int nb,
                                            WarpCols<F32>& sm, int lane, int topm, double zhi,
                                            double zlo, double (&acc)[6], int nd, double pm) {
  using W = typename WaSel<F32>::W;
  using R = typename WaSel<F32>::R;
  const R ig = (R)a.inv_gamma;
  constexpr int KM = D ? D : kMaxStagedDeg;
  const int DD = D ? D : nd;
  // z-cut phase first: its column is then recycled as the FD accumulator
  W wz;
  wz.init();
P3D_K1_LOOP_UNROLL
  for (int k = 0; k < DD; ++k) {
    R ep, em;
    W::term(sm.pz[k][lane], zhi, zlo, ig, ep, em);
    sm.ep[k][lane] = ep;
    sm.em[k][lane] = em;
    wz.acc(sm.pz[k][lane], zhi, zlo, ep, em, 1);
  }
  wz.finalize();
  acc[2] += pm * wz.value(zhi, zlo);
  const GradK<R> kz = wz.gk(zhi, zlo);
P3D_K1_LOOP_UNROLL
  for (int k = 0; k < DD; ++k) {
    sm.gc[k][lane] = (double)kz.grad(sm.pz[k][lane], ig, sm.ep[k][lane], sm.em[k][lane]);
    sm.pz[k][lane] = 0.0;
  }
  double v, ex;
  bool cross;
  int slot[KM];
  staged_axis<D, F32>(sm.px, sm, lane, topm, ig, v, ex, cross, nd);
  acc[0] += pm * v;
  acc[3] += pm * ex;
  acc[5] += pm * (cross ? 1.0 : 0.0);
  // the record slots load while the y axis is evaluated
#pragma unroll
  for (int k = 0; k < KM; ++k) {
    if (k >= DD) break;
    slot[k] = ld_stream(a.slot + pin0 + k * nb);
  }
  staged_axis<D, F32>(sm.py, sm, lane, topm, ig, v, ex, cross, nd);
  acc[1] += pm * v;
  acc[4] += pm * ex;
#pragma unroll
  for (int k = 0; k < KM; ++k) {
    if (k >= DD) break;
    const double dwk = sm.pz[k][lane];
    const double gb = (((topm >> k) & 1) ? -dwk : dwk) * a.scale4;
    if (F32)
      a.out_f[slot[k]] = make_float4((float)sm.px[k][lane], (float)sm.py[k][lane],
                                     (float)sm.gc[k][lane], (float)gb);
    else
      store_rec(a.out_d, slot[k], sm.px[k][lane], sm.py[k][lane], sm.gc[k][lane], gb);
  }
}

// Degree-3 nets (a fifth of all nets) are never split either — one die holds
// at most one pin or all three, so top + bot <= full — and their FD flip
// delta is exactly 0: flipping a pin leaves spans that are differences of the
// same coordinates and never exceed the full span (rounding is monotonic), so
// max(full, sp + op) - full = 0 (wirelength.py:227-248).  Register-resident
// like the pair path; the WA sums run in pin order as in the staged path (the
// per-net totals may associate differently: same values to the last ulp).
template <bool F32>
__device__ __forceinline__ void triple_axis(const double (&v)[3], typename WaSel<F32>::R ig,
                                            double& val, double (&g)[3]) {
  using W = typename WaSel<F32>::W;
  using R = typename WaSel<F32>::R;
  const double hi = dmax(dmax(v[0], v[1]), v[2]), lo = dmin(dmin(v[0], v[1]), v[2]);
  R ep[3], em[3];
  W w;
  w.init();
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    W::term(v[k], hi, lo, ig, ep[k], em[k]);
    w.acc(v[k], hi, lo, ep[k], em[k], 1);
  }
  w.finalize();
  val = w.value(hi, lo);
  const GradK<R> gk = w.gk(hi, lo);
#pragma unroll
  for (int k = 0; k < 3; ++k) g[k] = (double)gk.grad(v[k], ig, ep[k], em[k]);
}

template <bool F32>
__device__ __forceinline__ void triple_task(const FusedNetArgs& a, const int4 tk, int t0, int lane,
                                            double (&acc)[6]) {
  const int nb = tk.y, j = tk.z + lane;
  if (j >= nb) return;
  const uint8_t nd = a.net_dup[t0 + j];
#if !P3D_K1_EARLY
  if (nd & 1) return;  // duplicate-owner nets: generic kernel
#endif
  const double pm = (nd & 2) ? 0.0 : 1.0;  // value counted by another rank (halo mode)
  const int p0 = tk.x + j;
  int inst[3], slot[3];
  float4 off[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    inst[k] = ld_stream(a.pin_inst + p0 + k * nb);
    slot[k] = ld_stream(a.slot + p0 + k * nb);
    off[k] = ld_stream(a.off + p0 + k * nb);
  }
#if P3D_K1_EARLY
  if (nd & 1) return;  // duplicate-owner nets: generic kernel
#endif
  double x[3], y[3], z[3];
  int tp[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
#ifdef P3D_PROBE_NOGATHER
    const double4 q = a.pos4[inst[k] & 31];
#else
    const double4 q = a.pos4[inst[k]];
#endif
    tp[k] = (q.z - a.dz2) > 0.0;
    x[k] = q.x + (double)(tp[k] ? off[k].x : off[k].z);
    y[k] = q.y + (double)(tp[k] ? off[k].y : off[k].w);
    z[k] = q.z;
  }
  const typename WaSel<F32>::R ig = (typename WaSel<F32>::R)a.inv_gamma;
  double vx, vy, vz, gx[3], gy[3], gz[3];
  triple_axis<F32>(x, ig, vx, gx);
  triple_axis<F32>(y, ig, vy, gy);
  triple_axis<F32>(z, ig, vz, gz);
  acc[0] += pm * vx;
  acc[1] += pm * vy;
  acc[2] += pm * vz;
  acc[3] += pm * (dmax(dmax(x[0], x[1]), x[2]) - dmin(dmin(x[0], x[1]), x[2]));  // never split: full
  acc[4] += pm * (dmax(dmax(y[0], y[1]), y[2]) - dmin(dmin(y[0], y[1]), y[2]));
  const int ntop = tp[0] + tp[1] + tp[2];
  acc[5] += pm * ((ntop > 0 && ntop < 3) ? 1.0 : 0.0);
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    if (F32) a.out_f[slot[k]] = make_float4((float)gx[k], (float)gy[k], (float)gz[k], 0.f);
    else store_rec(a.out_d, slot[k], gx[k], gy[k], gz[k], 0.0);
  }
}

// Two-pin WA on one axis (wirelength.py:76-98): the anchor pin's terms are
// exp(0) = 1 and both non-trivial terms share the argument (lo - hi) / gamma,
// so one exponential serves the segment.  Accumulated exactly like the staged
// path (pin order), so the results are bit-identical to it.
template <bool F32>
__device__ __forceinline__ void pair_axis(double v0, double v1, typename WaSel<F32>::R ig,
                                          double& val, double& g0, double& g1) {
  using W = typename WaSel<F32>::W;
  using R = typename WaSel<F32>::R;
  const double hi = dmax(v0, v1), lo = dmin(v0, v1);
  const R e = W::gap(hi, lo, ig), one_p = (R)1, one_m = (R)1;  // exp((lo - hi)/g), exp(0)
  const bool first_hi = v0 >= v1;
  const R e0p = first_hi ? one_p : e, e1p = first_hi ? e : one_p;
  const R e0m = first_hi ? e : one_m, e1m = first_hi ? one_m : e;
  W w;
  w.init();
  w.acc(v0, hi, lo, e0p, e0m, 1);
  w.acc(v1, hi, lo, e1p, e1m, 1);
  w.finalize();
  val = w.value(hi, lo);
  g0 = (double)w.grad(v0, hi, lo, ig, e0p, e0m);
  g1 = (double)w.grad(v1, hi, lo, ig, e1p, e1m);
}

// Degree-2 nets (about half of all nets): never split (both partial spans are
// 0 or the full span) and the FD flip delta is exactly 0 for both pins
// (wirelength.py:227-248), so a lane evaluates its net from registers.
// One lane's degree-2 net: its loads, then its evaluation from registers.
struct PairLd {
  int ok, s0, s1;
  double pm;
  double2 q0, q1;  // (x, y) of the two owners
  double z0, z1;
  float4 o0, o1;
};

__device__ __forceinline__ PairLd pair_load(const FusedNetArgs& a, const int4 tk, int t0, int lane) {
  PairLd L;
  const int nb = tk.y, j = tk.z + lane;
  L.ok = 0;
  if (j >= nb) return L;
  const uint8_t nd = a.net_dup[t0 + j];
#if !P3D_K1_EARLY
  if (nd & 1) return L;  // duplicate-owner nets: generic kernel
#endif
  L.pm = (nd & 2) ? 0.0 : 1.0;  // value counted by another rank (halo mode)
  const int p0 = tk.x + j, p1 = p0 + nb;
  const int i0 = ld_stream(a.pin_inst + p0), i1 = ld_stream(a.pin_inst + p1);
  L.s0 = ld_stream(a.slot + p0);
  L.s1 = ld_stream(a.slot + p1);
  L.o0 = ld_stream(a.off + p0);
  L.o1 = ld_stream(a.off + p1);
#if P3D_K1_EARLY  // the flag load overlaps the pin loads instead of preceding them
  if (nd & 1) return L;  // duplicate-owner nets: generic kernel
#endif
#ifdef P3D_PROBE_NOGATHER
  const double* pb0 = reinterpret_cast<const double*>(a.pos4 + (i0 & 31));
  const double* pb1 = reinterpret_cast<const double*>(a.pos4 + (i1 & 31));
#else
  const double* pb0 = reinterpret_cast<const double*>(a.pos4 + i0);
  const double* pb1 = reinterpret_cast<const double*>(a.pos4 + i1);
#endif
  L.q0 = *reinterpret_cast<const double2*>(pb0);
  L.q1 = *reinterpret_cast<const double2*>(pb1);
  L.z0 = pb0[2];
  L.z1 = pb1[2];
  L.ok = 1;
  return L;
}

template <bool F32>
__device__ __forceinline__ void pair_eval(const FusedNetArgs& a, const PairLd& L, double (&acc)[6]) {
  if (!L.ok) return;
  const double2 q0 = L.q0, q1 = L.q1;
  const float4 o0 = L.o0, o1 = L.o1;
  const double pm = L.pm;
  const int t0p = (L.z0 - a.dz2) > 0.0, t1p = (L.z1 - a.dz2) > 0.0;
  const double x0 = q0.x + (double)(t0p ? o0.x : o0.z), y0 = q0.y + (double)(t0p ? o0.y : o0.w);
  const double x1 = q1.x + (double)(t1p ? o1.x : o1.z), y1 = q1.y + (double)(t1p ? o1.y : o1.w);
  const typename WaSel<F32>::R ig = (typename WaSel<F32>::R)a.inv_gamma;
  double vx, vy, vz, gx0, gx1, gy0, gy1, gz0, gz1;
  pair_axis<F32>(x0, x1, ig, vx, gx0, gx1);
  pair_axis<F32>(y0, y1, ig, vy, gy0, gy1);
  pair_axis<F32>(L.z0, L.z1, ig, vz, gz0, gz1);
  acc[0] += pm * vx;
  acc[1] += pm * vy;
  acc[2] += pm * vz;
  acc[3] += pm * (dmax(x0, x1) - dmin(x0, x1));
  acc[4] += pm * (dmax(y0, y1) - dmin(y0, y1));
  acc[5] += pm * ((t0p != t1p) ? 1.0 : 0.0);
  if (F32) {
    a.out_f[L.s0] = make_float4((float)gx0, (float)gy0, (float)gz0, 0.f);
    a.out_f[L.s1] = make_float4((float)gx1, (float)gy1, (float)gz1, 0.f);
  } else {
    store_rec(a.out_d, L.s0, gx0, gy0, gz0, 0.0);
    store_rec(a.out_d, L.s1, gx1, gy1, gz1, 0.0);
  }
}

// Degree-2 nets (about half of all nets): never split (both partial spans are
// 0 or the full span) and the FD flip delta is exactly 0 for both pins
// (wirelength.py:227-248), so a lane evaluates its net from registers.
template <bool F32>
__device__ __forceinline__ void pair_task(const FusedNetArgs& a, const int4 tk, int t0, int lane,
                                          double (&acc)[6]) {
  pair_eval<F32>(a, pair_load(a, tk, t0, lane), acc);
}


template <int D, bool F32>
__device__ __forceinline__ void staged_task(const FusedNetArgs& a, const int4 tk, int t0,
                                            WarpCols<F32>& sm, int lane, double (&acc)[6]) {
  const int nd = tk.w;
  int topm;
  double zhi, zlo, pm;
  if (stage_pins<D, F32>(a, tk, t0, sm, lane, topm, zhi, zlo, pm))
    staged_eval<D, F32>(a, tk.x + tk.z + lane, tk.y, sm, lane, topm, zhi, zlo, acc, nd, pm);
}


template <bool F32>
__global__ void __launch_bounds__(32 * kWarpsPerBlock, P3D_K1_MINB) fused_net_kernel(FusedNetArgs a) {
  extern __shared__ __align__(16) unsigned char dyn_smem[];
  __shared__ double red[32 * 6];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int wstride = gridDim.x * kWarpsPerBlock;
#if P3D_K1_EARLY  // the next task's descriptor is loaded while this one runs
  // (the first one before the grid wait: the task list is constant)
  int wn = a.task_rank + (blockIdx.x * kWarpsPerBlock + wib) * a.task_size;
  int4 tkn = make_int4(0, 0, 0, 0);
  int t0n = 0;
  if (wn < a.n_tasks) { tkn = __ldg(a.tasks + wn); t0n = __ldg(a.task_t0 + wn); }
#endif
  pdl_wait();
  if (a.halt && *a.halt) return;
  if (a.gamma_ptr) a.gamma = *a.gamma_ptr;
  a.inv_gamma = 1.0 / a.gamma;
  double acc[6] = {0, 0, 0, 0, 0, 0};
  WarpCols<F32>& sm = reinterpret_cast<WarpCols<F32>*>(dyn_smem)[wib];
#if P3D_K1_EARLY
  for (;;) {
    if (wn >= a.n_tasks) break;
    const int4 tk = tkn;
    const int t0 = t0n;
    wn += wstride * a.task_size;
    if (wn < a.n_tasks) { tkn = a.tasks[wn]; t0n = a.task_t0[wn]; }
#else
  for (int j = blockIdx.x * kWarpsPerBlock + wib;; j += wstride) {
    const int w = a.task_rank + j * a.task_size;  // this rank's warp tasks (sharded loop)
    if (w >= a.n_tasks) break;
    const int4 tk = a.tasks[w];
    const int t0 = a.task_t0[w];
#endif
    // timing probes only (they drop work; results are wrong): -DP3D_SKIP_D2 / _DGE3
#ifdef P3D_SKIP_D2
    if (tk.w == 2) continue;
#endif
#ifdef P3D_SKIP_DGE3
    if (tk.w >= 3) continue;
#endif
    switch (tk.w) {
      case 2: pair_task<F32>(a, tk, t0, lane, acc); break;
#if P3D_K1_TRIPLE
      case 3: triple_task<F32>(a, tk, t0, lane, acc); break;
#else
      case 3: staged_task<3, F32>(a, tk, t0, sm, lane, acc); break;
#endif
#if P3D_K1_RTD
      case 4: case 5: case 6: staged_task<0, F32>(a, tk, t0, sm, lane, acc); break;
#else
      case 4: staged_task<4, F32>(a, tk, t0, sm, lane, acc); break;
      case 5: staged_task<5, F32>(a, tk, t0, sm, lane, acc); break;
      case 6: staged_task<6, F32>(a, tk, t0, sm, lane, acc); break;
#endif
      default: break;  // generic nets run in generic_net_kernel
    }
  }
  block_sum<6>(acc, red);
  if (threadIdx.x == 0)
    for (int q = 0; q < 6; ++q) a.partials[q * gridDim.x + blockIdx.x] = acc[q];
  if (last_block(a.counter)) {
    double v[6];
    ordered_sums<6>(a.partials, gridDim.x, gridDim.x, red, v);
    if (threadIdx.x == 0)
      for (int q = 0; q < 6; ++q) a.final6[q] = a.n_generic ? v[q] + a.generic6[q] : v[q];
  }
}

// Nets of degree outside [2, kMaxStagedDeg] (none in the synthetic designs):
// thread per net, pins re-loaded per pass; totals in generic6 (added by the
// staged kernel's epilogue, so the reduction order stays fixed).
template <bool F32>
__global__ void __launch_bounds__(256) generic_net_kernel(FusedNetArgs a) {
  if (a.halt && *a.halt) return;
  __shared__ double red[32 * 6];
  if (a.gamma_ptr) a.gamma = *a.gamma_ptr;
  a.inv_gamma = 1.0 / a.gamma;
  double acc[6] = {0, 0, 0, 0, 0, 0};
  for (int j = blockIdx.x * blockDim.x + threadIdx.x;; j += gridDim.x * blockDim.x) {
    const int g = a.task_rank + j * a.task_size;  // this rank's generic nets (sharded loop)
    if (g >= a.n_generic) break;
    process_net_generic<F32>(a, a.generic_nets[g], acc);
  }
  block_sum<6>(acc, red);
  if (threadIdx.x == 0)
    for (int q = 0; q < 6; ++q) a.gpartials[q * gridDim.x + blockIdx.x] = acc[q];
  if (last_block(a.gcounter)) {
    for (int q = 0; q < 6; ++q) {
      const double v = ordered_sum(a.gpartials + q * gridDim.x, gridDim.x, red);
      if (threadIdx.x == 0) a.generic6[q] = v;
    }
  }
}

#ifndef P3D_GATHER_BATCH
#define P3D_GATHER_BATCH 4
#endif
constexpr int kGatherBatch = P3D_GATHER_BATCH;

// owner gather: per object, ordered fp64 sums over its contiguous slot records
// (pin order within the owner, like bincount)
__global__ void __launch_bounds__(256) fused_gather_kernel(FusedGatherArgs a) {
  pdl_wait();
  if (a.halt && *a.halt) return;
  __shared__ double red[32 * 3];
  double acc[3] = {0, 0, 0};
  const int stride = gridDim.x * blockDim.x;
  for (int il = blockIdx.x * blockDim.x + threadIdx.x; il < a.n_obj; il += stride) {
    const int i = a.obj0 + il;
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
    const int b = a.obj_slot_ptr[i], e = a.obj_slot_ptr[i + 1];
    if (a.in_d) {
      // the first kGatherBatch records are loaded together (predicated, no
      // branch between them), then summed in slot order: one memory round
      // trip for almost every object instead of one per record
      const double2* r2 = reinterpret_cast<const double2*>(a.in_d);
      double2 ra[kGatherBatch], rb[kGatherBatch];
#pragma unroll
      for (int k = 0; k < kGatherBatch; ++k) {
        if (b + k < e) {
          ra[k] = __ldcs(r2 + 2 * (long long)(b + k));  // dead after this read
          rb[k] = __ldcs(r2 + 2 * (long long)(b + k) + 1);
        }
      }
#pragma unroll
      for (int k = 0; k < kGatherBatch; ++k) {
        if (b + k < e) { s0 += ra[k].x; s1 += ra[k].y; s2 += rb[k].x; s3 += rb[k].y; }
      }
      for (int s = b + kGatherBatch; s < e; ++s) {
        const double2 xa = __ldcs(r2 + 2 * (long long)s), xb = __ldcs(r2 + 2 * (long long)s + 1);
        s0 += xa.x; s1 += xa.y; s2 += xb.x; s3 += xb.y;
      }
    } else {
#pragma unroll 4
      for (int s = b; s < e; ++s) {
        const float4 r = a.in_f[s];
        s0 += (double)r.x; s1 += (double)r.y; s2 += (double)r.z; s3 += (double)r.w;
      }
    }
    reinterpret_cast<double4*>(a.out)[i] = make_double4(s0, s1, s2, s3);  // [n_obj][4]
    acc[0] += fabs(s0);
    acc[1] += fabs(s1);
    acc[2] += fabs(s3);
  }
  block_sum<3>(acc, red);
  if (threadIdx.x == 0)
    for (int q = 0; q < 3; ++q) a.partials[q * gridDim.x + blockIdx.x] = acc[q];
  if (a.final_norms && last_block(a.counter)) {  // sharded loop: norms after the all-reduce
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

// Warp-cooperative variant (fp64 records): a warp owns 32 consecutive
// objects, whose records are one contiguous slot range; the warp copies the
// range into shared memory with coalesced 16-byte loads (all in flight
// together), then each lane sums its own object's records in slot order —
// the same order, hence the same values, as the thread-per-object kernel.
constexpr int kGatherWarps = 8;
constexpr int kGatherStage = 128;  // records staged per warp and chunk (4 KB)
__global__ void __launch_bounds__(32 * kGatherWarps) gather_warp_kernel(FusedGatherArgs a) {
  pdl_wait();
  if (a.halt && *a.halt) return;
  __shared__ double2 stage[kGatherWarps][2 * kGatherStage];
  __shared__ double red[32 * 3];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const double2* in2 = reinterpret_cast<const double2*>(a.in_d);
  double2* st = stage[wib];
  double acc[3] = {0, 0, 0};
  const int wstride = gridDim.x * kGatherWarps * 32;
  for (int o0 = (blockIdx.x * kGatherWarps + wib) * 32; o0 < a.n_obj; o0 += wstride) {
    const int il = o0 + lane, i = a.obj0 + il;
    const int last = min(a.n_obj, o0 + 32) - 1;
    const int b = il <= last ? a.obj_slot_ptr[i] : 0;
    const int e = il <= last ? a.obj_slot_ptr[i + 1] : 0;
    const int rb = __shfl_sync(0xffffffffu, b, 0);
    const int re = __shfl_sync(0xffffffffu, e, last - o0);
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
    for (int c0 = rb; c0 < re; c0 += kGatherStage) {
      const int c1 = min(re, c0 + kGatherStage), nv = 2 * (c1 - c0);
      __syncwarp();
#pragma unroll
      for (int k = 0; k < 2 * kGatherStage / 32; ++k) {
        const int t = lane + 32 * k;
        if (t < nv) st[t] = __ldcs(in2 + 2 * (long long)c0 + t);  // dead after this read
      }
      __syncwarp();
      const int lo = max(b, c0), hi = min(e, c1);
      for (int r = lo; r < hi; ++r) {
        const double2 ra = st[2 * (r - c0)], rb2 = st[2 * (r - c0) + 1];
        s0 += ra.x; s1 += ra.y; s2 += rb2.x; s3 += rb2.y;
      }
    }
    if (il <= last) {
      reinterpret_cast<double4*>(a.out)[i] = make_double4(s0, s1, s2, s3);  // [n_obj][4]
      acc[0] += fabs(s0);
      acc[1] += fabs(s1);
      acc[2] += fabs(s3);
    }
  }
  block_sum<3>(acc, red);
  if (threadIdx.x == 0)
    for (int q = 0; q < 3; ++q) a.partials[q * gridDim.x + blockIdx.x] = acc[q];
  if (a.final_norms && last_block(a.counter)) {
    double n[3];
    ordered_sums<3>(a.partials, gridDim.x, gridDim.x, red, n);
    if (threadIdx.x == 0) {
      a.final_norms[0] = n[0];
      a.final_norms[1] = n[1];
      a.final_norms[2] = n[2];
      a.final_norms[3] = n[2] == 0.0 ? 0.0 : (n[0] + n[1]) / (2.0 * n[2]);  // Eq. 17
    }
  }
}

}  // namespace

void fused_net_setup() {
  static bool done_dev[kMaxDevices] = {};  // function attributes are per device
  bool& done = done_dev[current_device()];
  if (done) return;
  cudaFuncSetAttribute(fused_net_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)(kWarpsPerBlock * sizeof(WarpCols<true>)));
  cudaFuncSetAttribute(fused_net_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)(kWarpsPerBlock * sizeof(WarpCols<false>)));
  done = true;
}

void launch_fused_net(const FusedNetArgs& a, bool f32, cudaStream_t s) {
  if (a.n_generic > 0) {
    const int gb = grid_blocks(a.n_generic, 256, kMaxBlocks);
    if (f32) generic_net_kernel<true><<<gb, 256, 0, s>>>(a);
    else generic_net_kernel<false><<<gb, 256, 0, s>>>(a);
  }
  if (f32)
    pdl_launch_tag(1, fused_net_kernel<true>, a.blocks, 32 * kWarpsPerBlock, kWarpsPerBlock * sizeof(WarpCols<true>), s, a);
  else
    pdl_launch_tag(1, fused_net_kernel<false>, a.blocks, 32 * kWarpsPerBlock, kWarpsPerBlock * sizeof(WarpCols<false>), s, a);
}

#ifndef P3D_GATHER_WARP
#define P3D_GATHER_WARP 1
#endif
void launch_fused_gather(const FusedGatherArgs& a, cudaStream_t s) {
  if (P3D_GATHER_WARP && a.in_d) {
    FusedGatherArgs w = a;  // one warp per 32 objects, same partial slots
    w.blocks = std::min(a.blocks, std::max(1, (a.n_obj + 32 * kGatherWarps - 1) / (32 * kGatherWarps)));
    pdl_launch_tag(2, gather_warp_kernel, w.blocks, 32 * kGatherWarps, 0, s, w);
    return;
  }
  pdl_launch_tag(2, fused_gather_kernel, a.blocks, 256, 0, s, a);
}

}  // namespace p3d
