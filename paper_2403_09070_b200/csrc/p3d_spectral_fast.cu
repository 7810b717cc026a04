// K3 fast path — the spectral solve in three kernels instead of six passes,
// for power-of-two nx, ny >= 8 and nz <= kMaxNz (every BASELINE config):
//   A  yz-forward : one x-slab [ny][nz] (contiguous) per CTA: int64 fixed-point
//                   rho -> float64 (+ overflow excess, + re-zero for the next
//                   scatter), DCT-II along z (direct, nz small) and along y
//                   (Makhoul FFT), written back as X_yz;
//   B  x          : a tile of C columns x all nx rows per CTA: DCT-II along x,
//                   then for each of the 4 outputs the spectral coefficient
//                   scaling (1/lambda, omega) and the inverse transform along x
//                   (cosine series for phi, Ey, Ez; sine series for Ex);
//   C  yz-inverse : one x-slab of each of the 4 maps per CTA: inverse along y
//                   and z, written as the interleaved [B][4] (phi, Ex, Ey, Ez)
//                   map the density gather reads.
// The math (Makhoul reorderings, coefficient scaling) is p3d_spectral.cu's;
// this file only changes how the passes are grouped (3 launches, each slab /
// tile read once).
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

// Pre-process nl real lines (element k of line l at r[l*rs + k*es]) into
// bit-reversed complex FFT input (Makhoul).  N = 2^logN: all index math is
// shifts and masks.
__device__ __forceinline__ void pre_lines(int op, const double* r, int rs, int es, int nl, int N,
                                          int logN, const double* ph, double2* c) {
  const int shift = 32 - logN;
  for (int t = threadIdx.x; t < (nl << logN); t += blockDim.x) {
    const int l = t >> logN, n = t & (N - 1);
    const double* line = r + l * rs;
    double2 v;
    int pos;
    if (op == T_DCT2) {
      pos = (n & 1) ? N - 1 - (n >> 1) : (n >> 1);
      v = make_double2(line[n * es], 0.0);
    } else {
      const int k = n;
      double ck, cn;
      if (op == T_COS) {
        ck = line[k * es];
        cn = k ? line[(N - k) * es] : 0.0;
      } else {
        ck = k ? line[(N - k) * es] : 0.0;
        cn = k ? line[k * es] : 0.0;
      }
      const double A = (k ? 0.5 : 1.0) * ck, B = 0.5 * cn;
      const double cs = ph[2 * k], sn = ph[2 * k + 1];
      v = make_double2(cs * A + sn * B, sn * A - cs * B);
      pos = k;
    }
    c[(l << logN) + (__brev(pos) >> shift)] = v;
  }
}

// in-place radix-2 DIT over nl lines (bit-reversed input, natural output);
// twiddles staged in shared memory by the caller (tw: N/2 complex)
__device__ __forceinline__ void fft_lines(double2* c, int nl, int N, int logN, const double2* tw,
                                          bool inv) {
  const int lhalf = logN - 1;
  for (int s = 0; s < logN; ++s) {
    const int half = 1 << s;
    for (int t = threadIdx.x; t < (nl << lhalf); t += blockDim.x) {
      const int l = t >> lhalf, b = t & ((1 << lhalf) - 1);
      const int j = b & (half - 1);
      const int i0 = ((b >> s) << (s + 1)) + j, i1 = i0 + half;
      double2 w = tw[j << (lhalf - s)];
      if (inv) w.y = -w.y;
      double2* buf = c + (l << logN);
      const double2 x0 = buf[i0], x1 = cmul(w, buf[i1]);
      buf[i0] = make_double2(x0.x + x1.x, x0.y + x1.y);
      buf[i1] = make_double2(x0.x - x1.x, x0.y - x1.y);
    }
    __syncthreads();
  }
}

// Post-process FFT output into real lines (element m at r[l*rs + m*es]).
__device__ __forceinline__ void post_lines(int op, const double2* c, int nl, int N, int logN,
                                           const double* ph, double* r, int rs, int es) {
  for (int t = threadIdx.x; t < (nl << logN); t += blockDim.x) {
    const int l = t >> logN, m = t & (N - 1);
    const double2* buf = c + (l << logN);
    double y;
    if (op == T_DCT2) {
      y = ph[2 * m] * buf[m].x + ph[2 * m + 1] * buf[m].y;
    } else {
      const int idx = (m & 1) ? N - 1 - (m >> 1) : (m >> 1);
      y = buf[idx].x;
      if (op == T_SIN && (m & 1)) y = -y;
    }
    r[l * rs + m * es] = y;
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
  double* M;              // [4][B] intermediate
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
  double* slab = sm;                                   // [S]
  double* tmp = sm + S;                                // [S]
  double2* cb = reinterpret_cast<double2*>(sm + 2 * S);  // [S] complex
  double2* tw = reinterpret_cast<double2*>(sm + 4 * S);  // [ny/2]
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
  pre_lines(T_DCT2, slab, 1, nz, nz, ny, a.logy, a.phy, cb);
  __syncthreads();
  fft_lines(cb, nz, ny, a.logy, tw, false);
  post_lines(T_DCT2, cb, nz, ny, a.logy, a.phy, slab, 1, nz);
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

// ---- B: x-lines of a C-column tile: DCT-II, then the 4 outputs' coefficient
// scaling + inverse transforms batched into one FFT pass of 4C lines.  Output
// M is interleaved [B][4] so kernel C reads whole slabs of all four maps.
__device__ __forceinline__ int col_tile(int nx) { return nx >= 1024 ? 1 : 1024 / nx; }

__global__ void __launch_bounds__(kThreads) spec_x(FastArgs a) {
  if (a.halt && *a.halt) return;
  extern __shared__ double sm[];
  const int nx = a.nx, S = a.ny * a.nz, C = col_tile(nx), lg = a.logx;
  const int c0 = blockIdx.x * C;
  double* X = sm;                                              // [C][nx]
  double* R = X + C * nx;                                      // [4C][nx]
  double2* cb = reinterpret_cast<double2*>(R + 4 * C * nx);    // [4C][nx]
  double2* tw = cb + 4 * C * nx;                               // [nx/2]
  stage_twiddles(a.twx, nx, tw);
  const double* src = a.coef_in ? a.coef_in : a.X;
  for (int t = threadIdx.x; t < C * nx; t += blockDim.x) {
    const int ix = t / C, c = t - ix * C;  // consecutive threads: consecutive columns
    X[c * nx + ix] = src[(long long)ix * S + c0 + c];
  }
  __syncthreads();
  if (!a.coef_in) {
    pre_lines(T_DCT2, X, nx, 1, C, nx, lg, a.phx, cb);
    __syncthreads();
    fft_lines(cb, C, nx, lg, tw, false);
    post_lines(T_DCT2, cb, C, nx, lg, a.phx, X, nx, 1);
    __syncthreads();
    if (a.coef_out)
      for (int t = threadIdx.x; t < C * nx; t += blockDim.x) {
        const int ix = t / C, c = t - ix * C;
        a.coef_out[(long long)ix * S + c0 + c] = 8.0 * X[c * nx + ix];
      }
  }
  if (!a.maps) return;
  // line L = map * C + c: scaled coefficients -> bit-reversed Makhoul input
  const int shift = 32 - lg;
  for (int t = threadIdx.x; t < (4 * C) << lg; t += blockDim.x) {
    const int L = t >> lg, k = t & (nx - 1);
    const int map = L / C, c = L - map * C;
    const int col = c0 + c, ky = col / a.nz, kz = col - ky * a.nz;
    const double* line = X + c * nx;
    const int kn = (nx - k) & (nx - 1);
    const double fk = coef_factor(a, k, ky, kz, map), fn = coef_factor(a, kn, ky, kz, map);
    double ck, cn;
    if (map != 1) {  // cosine series along x (phi, Ey, Ez)
      ck = line[k] * fk;
      cn = k ? line[kn] * fn : 0.0;
    } else {  // sine series along x (Ex)
      ck = k ? line[kn] * fn : 0.0;
      cn = k ? line[k] * fk : 0.0;
    }
    const double A = (k ? 0.5 : 1.0) * ck, B = 0.5 * cn;
    const double cs = a.phx[2 * k], sn = a.phx[2 * k + 1];
    cb[(L << lg) + (__brev(k) >> shift)] = make_double2(cs * A + sn * B, sn * A - cs * B);
  }
  __syncthreads();
  fft_lines(cb, 4 * C, nx, lg, tw, true);
  for (int t = threadIdx.x; t < (4 * C) << lg; t += blockDim.x) {
    const int L = t >> lg, m = t & (nx - 1);
    const int idx = (m & 1) ? nx - 1 - (m >> 1) : (m >> 1);
    double y = cb[(L << lg) + idx].x;
    if (L / C == 1 && (m & 1)) y = -y;
    R[t] = y;
  }
  __syncthreads();
  // interleaved write: for each row ix, C columns x 4 maps are contiguous
  for (int t = threadIdx.x; t < 4 * C * nx; t += blockDim.x) {
    const int ix = t / (4 * C), r = t - ix * 4 * C, c = r >> 2, map = r & 3;
    a.M[((long long)ix * S + c0 + c) * 4 + map] = R[((map * C + c) << lg) + ix];
  }
}

// ---- C: inverse along y then z for the 4 maps of one x-slab -> [B][4];
// the 4*nz y-lines of the slab are one FFT batch
__global__ void __launch_bounds__(kThreads) spec_inv_yz(FastArgs a) {
  if (a.halt && *a.halt) return;
  extern __shared__ double sm[];
  const int ny = a.ny, nz = a.nz, S = ny * nz, lg = a.logy;
  double* slab = sm;                                          // [4][S]
  double* tmp = slab + 4 * S;                                 // [S]
  double2* cb = reinterpret_cast<double2*>(tmp + S);          // [4 nz][ny]
  double2* tw = cb + 4 * S;                                   // [ny/2]
  stage_twiddles(a.twy, ny, tw);
  const long long base = (long long)blockIdx.x * S;
  for (int t = threadIdx.x; t < 4 * S; t += blockDim.x)  // contiguous interleaved slab
    slab[(t & 3) * S + (t >> 2)] = a.M[base * 4 + t];
  __syncthreads();
  // pre: line L = map * nz + iz, element iy at slab[map][iy*nz + iz]
  const int shift = 32 - lg;
  for (int t = threadIdx.x; t < (4 * nz) << lg; t += blockDim.x) {
    const int L = t >> lg, k = t & (ny - 1);
    const int map = L / nz, iz = L - map * nz;
    const double* line = slab + map * S + iz;
    const int kn = (ny - k) & (ny - 1);
    double ck, cn;
    if (map != 2) {  // cosine series along y (phi, Ex, Ez)
      ck = line[k * nz];
      cn = k ? line[kn * nz] : 0.0;
    } else {  // sine series along y (Ey)
      ck = k ? line[kn * nz] : 0.0;
      cn = k ? line[k * nz] : 0.0;
    }
    const double A = (k ? 0.5 : 1.0) * ck, B = 0.5 * cn;
    const double cs = a.phy[2 * k], sn = a.phy[2 * k + 1];
    cb[(L << lg) + (__brev(k) >> shift)] = make_double2(cs * A + sn * B, sn * A - cs * B);
  }
  __syncthreads();
  fft_lines(cb, 4 * nz, ny, lg, tw, true);
  for (int t = threadIdx.x; t < (4 * nz) << lg; t += blockDim.x) {
    const int L = t >> lg, m = t & (ny - 1);
    const int map = L / nz, iz = L - map * nz;
    const int idx = (m & 1) ? ny - 1 - (m >> 1) : (m >> 1);
    double y = cb[(L << lg) + idx].x;
    if (map == 2 && (m & 1)) y = -y;
    slab[map * S + m * nz + iz] = y;
  }
  __syncthreads();
  for (int map = 0; map < 4; ++map) z_direct(map == 3 ? T_SIN : T_COS, slab + map * S, ny, nz, tmp);
  for (int t = threadIdx.x; t < 4 * S; t += blockDim.x)
    a.maps[base * 4 + t] = slab[(t & 3) * S + (t >> 2)];
}

int ilog2_pow2(int n) {
  int l = 0;
  while ((1 << l) < n) ++l;
  return (1 << l) == n ? l : -1;
}

}  // namespace

constexpr size_t kSmemMax = 227 * 1024;
size_t smem_a(const p3d_grid* g) { return ((size_t)g->ny * g->nz * 4 + g->ny) * sizeof(double); }
size_t smem_b(const p3d_grid* g) {
  const size_t C = g->nx >= 1024 ? 1 : 1024 / g->nx;
  return (C * g->nx * (1 + 4 + 8) + g->nx) * sizeof(double);
}
size_t smem_c(const p3d_grid* g) {
  const size_t S = (size_t)g->ny * g->nz;
  return (4 * S + S + 8 * S + g->ny) * sizeof(double);
}

bool spectral_fast_ok(const p3d_grid* g) {
  const int lx = ilog2_pow2(g->nx), ly = ilog2_pow2(g->ny);
  return lx >= 3 && ly >= 3 && g->nz >= 1 && g->nz <= kMaxNz &&
         smem_a(g) <= kSmemMax && smem_b(g) <= kSmemMax && smem_c(g) <= kSmemMax &&
         g->nx <= 4096 && (g->ny * g->nz) % (g->nx >= 1024 ? 1 : 1024 / g->nx) == 0;
}

void spectral_fast_setup() {
  static bool done = false;
  if (done) return;
  cudaFuncSetAttribute(spec_fwd_yz, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemMax);
  cudaFuncSetAttribute(spec_x, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemMax);
  cudaFuncSetAttribute(spec_inv_yz, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemMax);
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
  const int C = g->nx >= 1024 ? 1 : 1024 / g->nx;
  spec_x<<<(int)(S / C), kThreads, smem_b(g), s>>>(a);
  if (maps) spec_inv_yz<<<g->nx, kThreads, smem_c(g), s>>>(a);
  return check_launch("spectral (fast path)");
}

}  // namespace p3d
