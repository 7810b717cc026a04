// K3 fast path — the spectral solve in three kernels instead of six passes,
// for power-of-two nx, ny >= 8 and nz <= kMaxNz (every BASELINE config):
//   A  yz-forward : one x-slab [ny][nz] (contiguous) per CTA: int64 fixed-point
//                   rho -> float64 (+ overflow excess, + re-zero for the next
//                   scatter), DCT-II along z (direct, nz small) and along y;
//   B  x          : one column x all nx rows per CTA: DCT-II along x, then the
//                   4 outputs' coefficient scaling (1/lambda, omega) and inverse
//                   transforms along x batched into one FFT pass (cosine series
//                   for phi, Ey, Ez; sine series for Ex), written interleaved;
//   C  yz-inverse : one x-slab of all 4 maps per CTA: inverse along y and z,
//                   written as the interleaved [B][4] (phi, Ex, Ey, Ez) map the
//                   density gather reads.
// Every 1-D transform is Makhoul's N-point complex FFT reordering (see
// p3d_spectral.cu for the math); the FFT itself is a self-sorting Stockham
// radix-4 (+ one radix-2 stage for odd log2 N) in shared memory, ping-ponging
// between two buffers: natural-order input and output, no bit reversal, and
// only the first one or two stages have strided (2-4 way conflicted) stores.
#include "p3d_common.cuh"
#include "p3d_internal.cuh"

namespace p3d {

namespace {

constexpr int kMaxNz = 16;
constexpr int kThreads = 256;

enum { T_DCT2 = 0, T_COS = 1, T_SIN = 2 };

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }

// e^{-2 pi i idx / N} from the half table tw[j] = e^{-2 pi i j / N}, j < N/2
__device__ __forceinline__ double2 twiddle(const double2* tw, int idx, int N, bool inv) {
  const int h = N >> 1;
  double2 w = idx < h ? tw[idx] : make_double2(-tw[idx - h].x, -tw[idx - h].y);
  if (inv) w.y = -w.y;
  return w;
}

// Stockham autosort FFT over nl lines of N = 2^logN (line l at A + l*N).
// Returns the buffer holding the natural-order result (A or B).
__device__ double2* fft_stockham(double2* A, double2* B, int nl, int logN, const double2* tw,
                                 bool inv) {
  const int N = 1 << logN;
  double2* in = A;
  double2* out = B;
  int lns = 0;  // log2 Ns
  if (logN & 1) {  // one radix-2 stage (Ns = 1)
    const int q = N >> 1;
    for (int t = threadIdx.x; t < nl * q; t += blockDim.x) {
      const int l = t >> (logN - 1), j = t & (q - 1);
      const double2* src = in + (l << logN);
      double2* dst = out + (l << logN);
      const double2 v0 = src[j], v1 = src[j + q];
      dst[2 * j] = cadd(v0, v1);
      dst[2 * j + 1] = csub(v0, v1);
    }
    __syncthreads();
    double2* tmp = in; in = out; out = tmp;
    lns = 1;
  }
  for (; lns < logN; lns += 2) {  // radix-4 stages
    const int Ns = 1 << lns, q = N >> 2, tstride = N >> (lns + 2);
    for (int t = threadIdx.x; t < nl * q; t += blockDim.x) {
      const int l = t >> (logN - 2), j = t & (q - 1);
      const double2* src = in + (l << logN);
      double2* dst = out + (l << logN);
      const int k = j & (Ns - 1);
      double2 v0 = src[j], v1 = src[j + q], v2 = src[j + 2 * q], v3 = src[j + 3 * q];
      if (k) {
        const int e = k * tstride;  // W_{4Ns}^{r k} = W_N^{r k N/(4 Ns)}
        v1 = cmul(v1, twiddle(tw, e, N, inv));
        v2 = cmul(v2, twiddle(tw, 2 * e, N, inv));
        v3 = cmul(v3, twiddle(tw, 3 * e, N, inv));
      }
      const double2 a0 = cadd(v0, v2), a1 = csub(v0, v2), a2 = cadd(v1, v3);
      const double2 d = csub(v1, v3);
      const double2 a3 = inv ? make_double2(-d.y, d.x) : make_double2(d.y, -d.x);  // +-i d
      const int o = ((j - k) << 2) + k;
      dst[o] = cadd(a0, a2);
      dst[o + Ns] = cadd(a1, a3);
      dst[o + 2 * Ns] = csub(a0, a2);
      dst[o + 3 * Ns] = csub(a1, a3);
    }
    __syncthreads();
    double2* tmp = in; in = out; out = tmp;
  }
  return in;
}

// Makhoul pre-processing of one element into natural-order FFT input at `pos`.
__device__ __forceinline__ void pre_elem(int op, int n, int N, double xn, double ck, double cn,
                                         const double* ph, double2& v, int& pos) {
  if (op == T_DCT2) {
    pos = (n & 1) ? N - 1 - (n >> 1) : (n >> 1);  // v[n/2] = x[n], v[N-1-(n-1)/2] = x[n]
    v = make_double2(xn, 0.0);
  } else {  // V_k = e^{i pi k/2N} (t_k c_k - i t_{N-k} c_{N-k}), t_0 = 1, t_k = 1/2
    const double A = (n ? 0.5 : 1.0) * ck, B = 0.5 * cn;
    const double cs = ph[2 * n], sn = ph[2 * n + 1];
    v = make_double2(cs * A + sn * B, sn * A - cs * B);
    pos = n;
  }
}

// Pre-process nl real lines (element k of line l at r[l*rs + k*es]).
__device__ __forceinline__ void pre_lines(int op, const double* r, int rs, int es, int nl,
                                          int logN, const double* ph, double2* c) {
  const int N = 1 << logN;
  for (int t = threadIdx.x; t < (nl << logN); t += blockDim.x) {
    const int l = t >> logN, n = t & (N - 1);
    const double* line = r + l * rs;
    double ck = 0.0, cn = 0.0, xn = 0.0;
    if (op == T_DCT2) xn = line[n * es];
    else if (op == T_COS) { ck = line[n * es]; cn = n ? line[(N - n) * es] : 0.0; }
    else { ck = n ? line[(N - n) * es] : 0.0; cn = n ? line[n * es] : 0.0; }
    double2 v;
    int pos;
    pre_elem(op, n, N, xn, ck, cn, ph, v, pos);
    c[(l << logN) + pos] = v;
  }
}

// Post-process natural-order FFT output of one line (element m).
__device__ __forceinline__ double post_elem(int op, const double2* buf, int m, int N,
                                            const double* ph) {
  if (op == T_DCT2) return ph[2 * m] * buf[m].x + ph[2 * m + 1] * buf[m].y;  // Re(e^{-i pi k/2N} V_k)
  const int idx = (m & 1) ? N - 1 - (m >> 1) : (m >> 1);
  const double y = buf[idx].x;
  return (op == T_SIN && (m & 1)) ? -y : y;  // sine series: (-1)^m cosine series of c'
}

__device__ __forceinline__ void post_lines(int op, const double2* c, int nl, int logN,
                                           const double* ph, double* r, int rs, int es) {
  const int N = 1 << logN;
  for (int t = threadIdx.x; t < (nl << logN); t += blockDim.x) {
    const int l = t >> logN, m = t & (N - 1);
    r[l * rs + m * es] = post_elem(op, c + (l << logN), m, N, ph);
  }
}

__device__ __forceinline__ void stage_twiddles(const double* tw, int N, double2* smem_tw) {
  for (int j = threadIdx.x; j < (N >> 1); j += blockDim.x)
    smem_tw[j] = make_double2(tw[2 * j], tw[2 * j + 1]);
}

// direct transform along z of every row of a slab [ny][nz] held in smem;
// nz == 2 (every BASELINE config) is a closed-form butterfly
__device__ __forceinline__ void z_direct(int op, double* slab, int ny, int nz, double* tmp) {
  if (nz == 2) {
    const double r2 = 0.70710678118654752440;  // cos(pi/4) = sin(pi/4)
    for (int iy = threadIdx.x; iy < ny; iy += blockDim.x) {
      const double x0 = slab[2 * iy], x1 = slab[2 * iy + 1];
      double y0, y1;
      if (op == T_DCT2) { y0 = x0 + x1; y1 = (x0 - x1) * r2; }
      else if (op == T_COS) { y0 = x0 + x1 * r2; y1 = x0 - x1 * r2; }
      else { y0 = x1 * r2; y1 = x1 * r2; }
      slab[2 * iy] = y0;
      slab[2 * iy + 1] = y1;
    }
    __syncthreads();
    return;
  }
  const int mod = 4 * nz;
  for (int t = threadIdx.x; t < ny * nz; t += blockDim.x) {
    const int iy = t / nz, m = t - iy * nz;
    const double* row = slab + iy * nz;
    double s = 0.0;
    for (int n = 0; n < nz; ++n) {
      const long long p = op == T_DCT2 ? (long long)m * (2 * n + 1) : (long long)n * (2 * m + 1);
      const double ang = (double)(p % mod) / (double)(2 * nz);
      if (op == T_SIN) {
        if (n) s += row[n] * sinpi(ang);
      } else {
        s += row[n] * cospi(ang);
      }
    }
    tmp[t] = s;
  }
  __syncthreads();
  for (int t = threadIdx.x; t < ny * nz; t += blockDim.x) slab[t] = tmp[t];
  __syncthreads();
}

struct FastArgs {
  int nx, ny, nz, logx, logy;
  const double *omx, *omy, *omz;
  const double *twx, *twy, *phx, *phy;
  const int64_t* rho_fx;  // A input (or rho_d)
  const double* rho_d;
  int64_t* zero_fx;       // nullable
  long long rho_t_fx;
  double* X;              // [B] intermediate
  double* M;              // [B][4] intermediate (interleaved)
  double* maps;           // [B][4] output
  const double* coef_in;  // nullable: B starts from scipy coef (electric_field)
  double in_scale;
  double* coef_out;       // nullable: scipy coef = 8 X
  double* partials;
  unsigned int* counter;
  double* ovfl_out;
  double ovfl_scale;
  const int* halt;
};

// ---- A: fixed-point rho -> X_yz (DCT-II along z, then y), overflow, re-zero
__global__ void __launch_bounds__(kThreads) spec_fwd_yz(FastArgs a) {
  if (a.halt && *a.halt) return;
  extern __shared__ double sm[];
  const int ny = a.ny, nz = a.nz, S = ny * nz;
  double* slab = sm;                                     // [S]
  double* tmp = sm + S;                                  // [S]
  double2* cA = reinterpret_cast<double2*>(sm + 2 * S);  // [S] complex
  double2* cB = cA + S;                                  // [S] complex
  double2* tw = cB + S;                                  // [ny/2]
  stage_twiddles(a.twy, ny, tw);
  const long long base = (long long)blockIdx.x * S;
  long long excess = 0;
  for (int t = threadIdx.x; t < S; t += blockDim.x) {
    double v;
    if (a.rho_fx) {
      const long long q = a.rho_fx[base + t];
      v = (double)q * 9.094947017729282379150390625e-13;  // 2^-40, exact
      const long long e = q - a.rho_t_fx;
      excess += e > 0 ? e : 0;
      if (a.zero_fx) a.zero_fx[base + t] = 0;
    } else {
      v = a.rho_d[base + t];
    }
    slab[t] = v;
  }
  __syncthreads();
  if (nz > 1) z_direct(T_DCT2, slab, ny, nz, tmp);
  // y lines: line iz, element iy at slab[iy*nz + iz]
  pre_lines(T_DCT2, slab, 1, nz, nz, a.logy, a.phy, cA);
  __syncthreads();
  const double2* res = fft_stockham(cA, cB, nz, a.logy, tw, false);
  post_lines(T_DCT2, res, nz, a.logy, a.phy, slab, 1, nz);
  __syncthreads();
  for (int t = threadIdx.x; t < S; t += blockDim.x) a.X[base + t] = slab[t];
  if (a.ovfl_out) {
    long long e = warp_sum_ll(excess);
    __shared__ long long ws[kThreads / 32];
    if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = e;
    __syncthreads();
    if (threadIdx.x == 0) {
      long long b = 0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) b += ws[w];
      reinterpret_cast<long long*>(a.partials)[blockIdx.x] = b;
    }
    if (last_block(a.counter)) {
      const long long s = block_sum_ll_partials(
          reinterpret_cast<const volatile long long*>(a.partials), gridDim.x);
      if (threadIdx.x == 0) *a.ovfl_out = (double)s * a.ovfl_scale;
    }
  }
}

// spectral coefficient of output map m at mode (j, k, l) (see p3d_spectral.cu)
__device__ __forceinline__ double coef_factor(const FastArgs& a, int j, int k, int l, int map) {
  const double ox = a.omx[j], oy = a.omy[k], oz = a.omz[l];
  const double lam = ox * ox + oy * oy + oz * oz;
  const double inv = lam > 0.0 ? 1.0 / lam : 0.0;
  double s = (j ? 2.0 : 1.0) / a.nx * ((k ? 2.0 : 1.0) / a.ny) * ((l ? 2.0 : 1.0) / a.nz) * inv;
  if (map == 1) s *= ox;
  else if (map == 2) s *= oy;
  else if (map == 3) s *= oz;
  return s * a.in_scale;
}

// ---- B: one x-column per CTA: DCT-II, then the 4 outputs' coefficient
// scaling + inverse transforms as one batched FFT of 4 lines.
__global__ void __launch_bounds__(kThreads) spec_x(FastArgs a) {
  if (a.halt && *a.halt) return;
  extern __shared__ double sm[];
  const int nx = a.nx, S = a.ny * a.nz, lg = a.logx;
  const int col = blockIdx.x, ky = col / a.nz, kz = col - ky * a.nz;
  double* X = sm;                                              // [nx]
  double* R = X + nx;                                          // [4][nx]
  double2* cA = reinterpret_cast<double2*>(R + 4 * nx);       // [4][nx]
  double2* cB = cA + 4 * nx;                                   // [4][nx]
  double2* tw = cB + 4 * nx;                                   // [nx/2]
  stage_twiddles(a.twx, nx, tw);
  const double* src = a.coef_in ? a.coef_in : a.X;
  for (int ix = threadIdx.x; ix < nx; ix += blockDim.x) X[ix] = src[(long long)ix * S + col];
  __syncthreads();
  if (!a.coef_in) {
    pre_lines(T_DCT2, X, nx, 1, 1, lg, a.phx, cA);
    __syncthreads();
    const double2* res = fft_stockham(cA, cB, 1, lg, tw, false);
    post_lines(T_DCT2, res, 1, lg, a.phx, X, nx, 1);
    __syncthreads();
    if (a.coef_out)
      for (int ix = threadIdx.x; ix < nx; ix += blockDim.x)
        a.coef_out[(long long)ix * S + col] = 8.0 * X[ix];
  }
  if (!a.maps) return;
  for (int t = threadIdx.x; t < 4 << lg; t += blockDim.x) {
    const int map = t >> lg, k = t & (nx - 1), kn = (nx - k) & (nx - 1);
    const double fk = coef_factor(a, k, ky, kz, map), fn = coef_factor(a, kn, ky, kz, map);
    double ck, cn;
    if (map != 1) { ck = X[k] * fk; cn = k ? X[kn] * fn : 0.0; }   // cosine series (phi, Ey, Ez)
    else { ck = k ? X[kn] * fn : 0.0; cn = k ? X[k] * fk : 0.0; }  // sine series (Ex)
    double2 v;
    int pos;
    pre_elem(T_COS, k, nx, 0.0, ck, cn, a.phx, v, pos);
    cA[(map << lg) + pos] = v;
  }
  __syncthreads();
  const double2* res = fft_stockham(cA, cB, 4, lg, tw, true);
  for (int t = threadIdx.x; t < 4 << lg; t += blockDim.x) {
    const int map = t >> lg, m = t & (nx - 1);
    R[t] = post_elem(map == 1 ? T_SIN : T_COS, res + (map << lg), m, nx, a.phx);
  }
  __syncthreads();
  for (int t = threadIdx.x; t < 4 * nx; t += blockDim.x) {  // 32-byte record per row
    const int ix = t >> 2, map = t & 3;
    a.M[((long long)ix * S + col) * 4 + map] = R[(map << lg) + ix];
  }
}

// ---- C: inverse along y then z for the 4 maps of one x-slab -> [B][4]
// (two FFT batches of 2*nz lines)
__global__ void __launch_bounds__(kThreads) spec_inv_yz(FastArgs a) {
  if (a.halt && *a.halt) return;
  extern __shared__ double sm[];
  const int ny = a.ny, nz = a.nz, S = ny * nz, SP = S + 1, lg = a.logy;
  double* slab = sm;                                          // [4][S+1] (padded)
  double* tmp = slab + 4 * SP;                                // [S]
  double2* cA = reinterpret_cast<double2*>(tmp + S);          // [2 nz][ny]
  double2* cB = cA + 2 * S;                                   // [2 nz][ny]
  double2* tw = cB + 2 * S;                                   // [ny/2]
  stage_twiddles(a.twy, ny, tw);
  const long long base = (long long)blockIdx.x * S;
  for (int t = threadIdx.x; t < 4 * S; t += blockDim.x)  // contiguous interleaved slab
    slab[(t & 3) * SP + (t >> 2)] = a.M[base * 4 + t];
  __syncthreads();
  for (int half = 0; half < 2; ++half) {
    // line L = mm * nz + iz (mm = 0, 1 -> map 2*half + mm), element iy at slab[map][iy*nz + iz]
    for (int t = threadIdx.x; t < (2 * nz) << lg; t += blockDim.x) {
      const int L = t >> lg, k = t & (ny - 1);
      const int mm = L / nz, iz = L - mm * nz, map = 2 * half + mm;
      const double* line = slab + map * SP + iz;
      const int kn = (ny - k) & (ny - 1);
      double ck, cn;
      if (map != 2) { ck = line[k * nz]; cn = k ? line[kn * nz] : 0.0; }  // cosine (phi, Ex, Ez)
      else { ck = k ? line[kn * nz] : 0.0; cn = k ? line[k * nz] : 0.0; }  // sine (Ey)
      double2 v;
      int pos;
      pre_elem(T_COS, k, ny, 0.0, ck, cn, a.phy, v, pos);
      cA[(L << lg) + pos] = v;
    }
    __syncthreads();
    const double2* res = fft_stockham(cA, cB, 2 * nz, lg, tw, true);
    for (int t = threadIdx.x; t < (2 * nz) << lg; t += blockDim.x) {
      const int L = t >> lg, m = t & (ny - 1);
      const int mm = L / nz, iz = L - mm * nz, map = 2 * half + mm;
      slab[map * SP + m * nz + iz] =
          post_elem(map == 2 ? T_SIN : T_COS, res + (L << lg), m, ny, a.phy);
    }
    __syncthreads();
  }
  for (int map = 0; map < 4; ++map)
    z_direct(map == 3 ? T_SIN : T_COS, slab + map * SP, ny, nz, tmp);
  for (int t = threadIdx.x; t < 4 * S; t += blockDim.x)
    a.maps[base * 4 + t] = slab[(t & 3) * SP + (t >> 2)];
}

int ilog2_pow2(int n) {
  int l = 0;
  while ((1 << l) < n) ++l;
  return (1 << l) == n ? l : -1;
}

constexpr size_t kSmemMax = 220 * 1024;  // opt-in limit is 227 KB minus static smem
size_t smem_a(const p3d_grid* g) {
  const size_t S = (size_t)g->ny * g->nz;
  return (2 * S + 4 * S + g->ny) * sizeof(double);
}
size_t smem_b(const p3d_grid* g) { return ((size_t)g->nx * (1 + 4 + 16) + g->nx) * sizeof(double); }
size_t smem_c(const p3d_grid* g) {
  const size_t S = (size_t)g->ny * g->nz;
  return (4 * (S + 1) + S + 8 * S + g->ny) * sizeof(double);
}

}  // namespace

bool spectral_fast_ok(const p3d_grid* g) {
  const int lx = ilog2_pow2(g->nx), ly = ilog2_pow2(g->ny);
  return lx >= 3 && ly >= 3 && g->nz >= 1 && g->nz <= kMaxNz && smem_a(g) <= kSmemMax &&
         smem_b(g) <= kSmemMax && smem_c(g) <= kSmemMax;
}

void spectral_fast_setup() {
  static bool done = false;
  if (done) return;
  if (cudaFuncSetAttribute(spec_fwd_yz, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemMax) ||
      cudaFuncSetAttribute(spec_x, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemMax) ||
      cudaFuncSetAttribute(spec_inv_yz, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemMax)) {
    set_error("spectral: cannot opt into %zu bytes of shared memory", kSmemMax);
    cudaGetLastError();
    return;
  }
  done = true;
}

int launch_spectral_fast(const p3d_grid* g, const double* rho, const int64_t* rho_fx,
                         const double* coef_in, double* coef_out, double* maps, double* scratch,
                         const int* halt, const SpecOvfl* ov, cudaStream_t s) {
  spectral_fast_setup();
  const long long S = (long long)g->ny * g->nz, B = g->nx * S;
  FastArgs a{};
  a.nx = g->nx; a.ny = g->ny; a.nz = g->nz;
  a.logx = ilog2_pow2(g->nx);
  a.logy = ilog2_pow2(g->ny);
  a.omx = g->omega[0]; a.omy = g->omega[1]; a.omz = g->omega[2];
  a.twx = g->twiddle[0]; a.twy = g->twiddle[1];
  a.phx = g->phase[0]; a.phy = g->phase[1];
  a.rho_fx = rho_fx;
  a.rho_d = rho;
  a.X = scratch;
  a.M = scratch + B;
  a.maps = maps;
  a.coef_in = coef_in;
  a.in_scale = coef_in ? 0.125 : 1.0;
  a.coef_out = coef_out;
  a.halt = halt;
  if (ov && rho_fx) {
    a.zero_fx = ov->zero ? const_cast<int64_t*>(rho_fx) : nullptr;
    a.rho_t_fx = ov->rho_t_fx;
    a.partials = ov->partials;
    a.counter = ov->counter;
    a.ovfl_out = ov->out;
    a.ovfl_scale = ov->scale;
  }
  if (!coef_in) spec_fwd_yz<<<g->nx, kThreads, smem_a(g), s>>>(a);
  spec_x<<<(int)S, kThreads, smem_b(g), s>>>(a);
  if (maps) spec_inv_yz<<<g->nx, kThreads, smem_c(g), s>>>(a);
  return check_launch("spectral (fast path)");
}

}  // namespace p3d
