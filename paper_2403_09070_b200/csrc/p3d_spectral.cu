// K3 — spectral Poisson solve and electric field (density.py:319-368).
//
// All four output maps are 3D cosine/sine series of ONE coefficient array
//   A_jkl = X_jkl * (w_j/nx)(w_k/ny)(w_l/nz) * inv_lam_jkl,   w_0 = 1, w_k>0 = 2,
// where X = DCT-II(rho) without scipy's per-axis factor 2 (scipy's coef = 8 X):
//   phi = C_x C_y C_z [A]                (== idctn(coef*inv_lam))
//   Ex  = S_x C_y C_z [A * omega_x]      (== _eval_cos(_eval_cos(_eval_sin)))
//   Ey  = C_x S_y C_z [A * omega_y]
//   Ez  = C_x C_y S_z [A * omega_z]
// with C: y_m = sum_k c_k cos(pi k (2m+1) / 2N) and S: the same with sin.
// Each 1-D pass is a batch of line transforms in shared memory: a radix-2 FFT
// (Makhoul's N-point reordering) for power-of-two N >= 8, a direct sum
// otherwise.  fp64 throughout (TF32 breaks trajectory parity);
// the maps are small enough (<= 17 MB at 1024^2 x 2) to stay L2-resident.
// Passes: fwd z (reads the int64 fixed-point rho, also the overflow excess and
// re-zeroes rho for the next scatter), fwd y, fwd x (in place), inverse x
// (4 maps, coefficient scaling fused into the load), inverse y, inverse z
// (writes the interleaved [B][4] map that the density gather reads).
#include <stdio.h>
#include <stdlib.h>

#include "p3d_common.cuh"
#include "p3d_internal.cuh"

namespace p3d {

enum LineOp { OP_DCT2 = 0, OP_COS = 1, OP_SIN = 2 };
enum LoadMode { LOAD_D = 0, LOAD_FX = 1, LOAD_SPEC = 2 };
enum StoreMode { STORE_D = 0, STORE_MAPS = 1 };

struct PassArgs {
  int N, logN, n_lines, lpb;
  long long q, A, B, stride;  // base(line) = (line / q) * A + (line % q) * B
  int load, store;
  int op[4];                  // per map (blockIdx.y)
  const double* in;           // + map * map_stride_in
  const int64_t* in_fx;
  long long map_stride_in;
  double* out;                // + map * map_stride_out (STORE_D)
  long long map_stride_out;
  double out_scale;
  // spectral factor (LOAD_SPEC)
  int nx, ny, nz;
  const double *wx, *wy, *wz;
  double in_scale;
  // tables for this axis
  const double* tw;   // [N/2] (cos, -sin)(2 pi j / N) interleaved
  const double* ph;   // [N]   (cos, sin)(pi k / 2N) interleaved
  // fused overflow + re-zero (LOAD_FX)
  int64_t* fx_zero;   // nullable: store 0 after reading
  long long rho_t_fx;
  double* partials;
  unsigned int* counter;
  double* ovfl_out;   // nullable
  double ovfl_scale;  // 2^-40 * bin_vol / movable_volume
  const int* halt;
};

__device__ __forceinline__ double spec_factor(const PassArgs& a, long long f, int map) {
  const long long yz = (long long)a.ny * a.nz;
  const int j = (int)(f / yz);
  const int k = (int)((f / a.nz) % a.ny);
  const int l = (int)(f % a.nz);
  const double ox = a.wx[j], oy = a.wy[k], oz = a.wz[l];
  const double lam = ox * ox + oy * oy + oz * oz;
  const double inv = lam > 0.0 ? 1.0 / lam : 0.0;
  double s = (j ? 2.0 : 1.0) / a.nx * ((k ? 2.0 : 1.0) / a.ny) * ((l ? 2.0 : 1.0) / a.nz) * inv;
  if (map == 1) s *= ox;
  else if (map == 2) s *= oy;
  else if (map == 3) s *= oz;
  return s * a.in_scale;
}

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}

__global__ void __launch_bounds__(256) line_pass(PassArgs a) {
  if (a.halt && *a.halt) return;
  extern __shared__ double smem[];
  const int N = a.N, L = a.lpb, map = blockIdx.y, op = a.op[map];
  const int line0 = blockIdx.x * L;
  const int nl = min(L, a.n_lines - line0);
  double* rbuf = smem;                                    // [L][N]
  double2* cbuf = reinterpret_cast<double2*>(smem + L * N);  // [L][N]
  const double* in = a.in ? a.in + map * a.map_stride_in : nullptr;
  const bool fft = a.logN >= 3 && (1 << a.logN) == N;
  long long excess = 0;

  // ---- load (coalesced: lines fastest when stride > 1, elements fastest otherwise)
  const int tot = nl * N;
  for (int t = threadIdx.x; t < tot; t += blockDim.x) {
    int l, n;
    if (a.stride == 1) { l = t / N; n = t - l * N; } else { n = t / nl; l = t - n * nl; }
    const int line = line0 + l;
    const long long f = (line / a.q) * a.A + (line % a.q) * a.B + (long long)n * a.stride;
    double v;
    if (a.load == LOAD_FX) {
      long long q = a.in_fx[f];
      v = (double)q * 9.094947017729282379150390625e-13;  // 2^-40, exact
      long long e = q - a.rho_t_fx;
      excess += e > 0 ? e : 0;
      if (a.fx_zero) a.fx_zero[f] = 0;
    } else {
      v = in[f];
      if (a.load == LOAD_SPEC) v *= spec_factor(a, f, map);
    }
    rbuf[l * N + n] = v;
  }
  __syncthreads();

  if (fft) {
    // ---- pre-process into bit-reversed complex input
    const int shift = 32 - a.logN;
    for (int t = threadIdx.x; t < tot; t += blockDim.x) {
      const int l = t / N, n = t - l * N;
      const double* r = rbuf + l * N;
      double2 val;
      int pos;
      if (op == OP_DCT2) {
        // Makhoul: v[n/2] = x[n] (n even), v[N-1-(n-1)/2] = x[n] (n odd)
        pos = (n & 1) ? N - 1 - (n >> 1) : (n >> 1);
        val = make_double2(r[n], 0.0);
      } else {
        // V_k = e^{i pi k/2N} (t_k c_k - i t_{N-k} c_{N-k}), t_0 = 1, t_k = 1/2
        const int k = n;
        double ck, cn;
        if (op == OP_COS) {
          ck = r[k];
          cn = k ? r[N - k] : 0.0;
        } else {  // sine series == (-1)^m * cosine series of c'_j = c_{N-j}, c'_0 = 0
          ck = k ? r[N - k] : 0.0;
          cn = k ? r[k] : 0.0;
        }
        const double A = (k ? 0.5 : 1.0) * ck, B = 0.5 * cn;
        const double c = a.ph[2 * k], s = a.ph[2 * k + 1];
        val = make_double2(c * A + s * B, s * A - c * B);
        pos = k;
      }
      cbuf[l * N + (__brev(pos) >> shift)] = val;
    }
    __syncthreads();
    // ---- radix-2 DIT, forward for DCT2, inverse (conjugate twiddles) otherwise
    const double sgn = op == OP_DCT2 ? 1.0 : -1.0;
    const int half_n = N >> 1;
    for (int len = 2; len <= N; len <<= 1) {
      const int half = len >> 1, tstep = N / len;
      for (int t = threadIdx.x; t < nl * half_n; t += blockDim.x) {
        const int l = t / half_n, b = t - l * half_n;
        const int grp = b / half, j = b - grp * half;
        const int i0 = grp * len + j, i1 = i0 + half;
        double2 w = make_double2(a.tw[2 * j * tstep], sgn * a.tw[2 * j * tstep + 1]);
        double2* buf = cbuf + l * N;
        double2 x0 = buf[i0], x1 = cmul(w, buf[i1]);
        buf[i0] = make_double2(x0.x + x1.x, x0.y + x1.y);
        buf[i1] = make_double2(x0.x - x1.x, x0.y - x1.y);
      }
      __syncthreads();
    }
    // ---- post-process back into rbuf (real outputs)
    for (int t = threadIdx.x; t < tot; t += blockDim.x) {
      const int l = t / N, m = t - l * N;
      const double2* buf = cbuf + l * N;
      double y;
      if (op == OP_DCT2) {
        const double c = a.ph[2 * m], s = a.ph[2 * m + 1];
        y = c * buf[m].x + s * buf[m].y;  // Re(e^{-i pi k/2N} V_k)
      } else {
        const int idx = (m & 1) ? N - 1 - (m >> 1) : (m >> 1);
        y = buf[idx].x;
        if (op == OP_SIN && (m & 1)) y = -y;
      }
      rbuf[l * N + m] = y;
    }
    __syncthreads();
  } else {
    // ---- direct O(N^2) sums (small or non-power-of-two N); exact angle reduction
    double* obuf = reinterpret_cast<double*>(cbuf);
    const int mod = 4 * N;
    for (int t = threadIdx.x; t < tot; t += blockDim.x) {
      const int l = t / N, m = t - l * N;
      const double* r = rbuf + l * N;
      double s = 0.0;
      for (int n = 0; n < N; ++n) {
        // DCT2: angle pi*m*(2n+1)/2N ; COS/SIN: pi*n*(2m+1)/2N
        const long long p = op == OP_DCT2 ? (long long)m * (2 * n + 1) : (long long)n * (2 * m + 1);
        const double ang = (double)(p % mod) / (double)(2 * N);
        if (op == OP_SIN) {
          if (n) s += r[n] * sinpi(ang);
        } else {
          s += r[n] * cospi(ang);
        }
      }
      obuf[l * N + m] = s;
    }
    __syncthreads();
    for (int t = threadIdx.x; t < tot; t += blockDim.x) rbuf[t] = obuf[t];
    __syncthreads();
  }

  // ---- store
  for (int t = threadIdx.x; t < tot; t += blockDim.x) {
    int l, n;
    if (a.stride == 1) { l = t / N; n = t - l * N; } else { n = t / nl; l = t - n * nl; }
    const int line = line0 + l;
    const long long f = (line / a.q) * a.A + (line % a.q) * a.B + (long long)n * a.stride;
    const double v = rbuf[l * N + n] * a.out_scale;
    if (a.store == STORE_MAPS) a.out[f * 4 + map] = v;
    else a.out[map * a.map_stride_out + f] = v;
  }

  if (a.load == LOAD_FX && a.ovfl_out) {
    // deterministic integer reduction of the overflow excess
    long long e = warp_sum_ll(excess);
    __shared__ long long wsum[32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (lane == 0) wsum[wid] = e;
    __syncthreads();
    if (threadIdx.x == 0) {
      long long b = 0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) b += wsum[w];
      reinterpret_cast<long long*>(a.partials)[blockIdx.x] = b;
    }
    if (last_block(a.counter)) {
      const long long s = block_sum_ll_partials(
          reinterpret_cast<const volatile long long*>(a.partials), gridDim.x);
      if (threadIdx.x == 0) *a.ovfl_out = (double)s * a.ovfl_scale;
    }
  }
}

// ---------------------------------------------------------------------------
// Opt the line-pass kernel into large dynamic shared memory.  Called from the
// non-captured entry points (init / per-op) so graph capture never sees it.
void spectral_setup() {
  spectral_fast_setup();
  static bool done_dev[kMaxDevices] = {};  // function attributes are per device
  bool& done = done_dev[current_device()];
  if (!done) {
    cudaFuncSetAttribute(line_pass, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    done = true;
  }
}

static int choose_lpb(int N, int n_lines) {
  int lpb = N >= 256 ? 4 : (N >= 64 ? 8 : 2048 / (N > 0 ? N : 1));
  if (lpb < 1) lpb = 1;
  if (lpb > 256) lpb = 256;
  if (lpb > n_lines) lpb = n_lines;
  return lpb;
}

static int ilog2_exact(int n) {
  int l = 0;
  while ((1 << l) < n) ++l;
  return ((1 << l) == n) ? l : -1;
}

static int run_pass(PassArgs a, int axis, const p3d_grid* g, int nmaps, cudaStream_t s) {
  const int nx = g->nx, ny = g->ny, nz = g->nz;
  if (axis == 0) { a.N = nx; a.n_lines = ny * nz; a.q = (long long)ny * nz; a.A = 0; a.B = 1; a.stride = (long long)ny * nz; }
  if (axis == 1) { a.N = ny; a.n_lines = nx * nz; a.q = nz; a.A = (long long)ny * nz; a.B = 1; a.stride = nz; }
  if (axis == 2) { a.N = nz; a.n_lines = nx * ny; a.q = 1; a.A = nz; a.B = 0; a.stride = 1; }
  a.logN = ilog2_exact(a.N);
  a.lpb = choose_lpb(a.N, a.n_lines);
  a.tw = g->twiddle[axis];
  a.ph = g->phase[axis];
  const size_t smem = (size_t)a.lpb * a.N * (sizeof(double) + 2 * sizeof(double));
  if (smem > 200 * 1024) {
    set_error("spectral: line length %d too large for one CTA", a.N);
    return P3D_ERR_UNSUPPORTED;
  }
  spectral_setup();
  dim3 grid((a.n_lines + a.lpb - 1) / a.lpb, nmaps);
  line_pass<<<grid, 256, smem, s>>>(a);
  return check_launch("spectral line pass");
}

__global__ void scale_copy_kernel(const double* in, double* out, long long n, double s) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    out[i] = in[i] * s;
}

void launch_scale_copy(const double* in, double* out, long long n, double s, cudaStream_t st) {
  int blocks = (int)((n + 255) / 256);
  if (blocks > 4096) blocks = 4096;
  if (blocks < 1) blocks = 1;
  scale_copy_kernel<<<blocks, 256, 0, st>>>(in, out, n, s);
}

int launch_spectral(const p3d_grid* g, const double* rho, const int64_t* rho_fx,
                    const double* coef_in, double* coef_out, double* maps, double* scratch,
                    const int* halt, cudaStream_t s) {
  return launch_spectral_ex(g, rho, rho_fx, coef_in, coef_out, maps, scratch, halt, nullptr, s);
}

int launch_spectral_ex(const p3d_grid* g, const double* rho, const int64_t* rho_fx,
                       const double* coef_in, double* coef_out, double* maps, double* scratch,
                       const int* halt, const SpecOvfl* ov, cudaStream_t s) {
  if (spectral_fast_ok(g) && !getenv("P3D_SPECTRAL_GENERIC"))
    return launch_spectral_fast(g, rho, rho_fx, coef_in, coef_out, maps, scratch, halt, ov, s);
  const long long B = (long long)g->nx * g->ny * g->nz;
  double* X = scratch;       // [B]
  double* M = scratch + B;   // [4][B]
  PassArgs a{};
  a.halt = halt;
  a.nx = g->nx; a.ny = g->ny; a.nz = g->nz;
  a.wx = g->omega[0]; a.wy = g->omega[1]; a.wz = g->omega[2];
  a.out_scale = 1.0;
  a.in_scale = 1.0;
  int rc;
  if (coef_in == nullptr) {
    // forward: z (from rho / rho_fx), y, x, all into X
    PassArgs f = a;
    f.op[0] = OP_DCT2;
    f.store = STORE_D;
    f.out = X;
    if (rho_fx) {
      f.load = LOAD_FX;
      f.in_fx = rho_fx;
      if (ov) {
        f.fx_zero = ov->zero ? const_cast<int64_t*>(rho_fx) : nullptr;
        f.rho_t_fx = ov->rho_t_fx;
        f.partials = ov->partials;
        f.counter = ov->counter;
        f.ovfl_out = ov->out;
        f.ovfl_scale = ov->scale;
      }
    } else {
      f.load = LOAD_D;
      f.in = rho;
    }
    if ((rc = run_pass(f, 2, g, 1, s))) return rc;
    f.load = LOAD_D; f.in = X; f.fx_zero = nullptr; f.ovfl_out = nullptr;
    if ((rc = run_pass(f, 1, g, 1, s))) return rc;
    if ((rc = run_pass(f, 0, g, 1, s))) return rc;
    if (coef_out) {
      // scipy's unnormalised dctn carries a factor 2 per axis: coef = 8 X
      launch_scale_copy(X, coef_out, B, 8.0, s);
      if ((rc = check_launch("coef copy"))) return rc;
    }
  }
  if (maps == nullptr) return P3D_OK;
  // inverse: x (4 maps, scaled coefficients), y, z -> interleaved maps
  PassArgs v = a;
  v.load = LOAD_SPEC;
  v.in = coef_in ? coef_in : X;
  v.in_scale = coef_in ? 0.125 : 1.0;
  v.map_stride_in = 0;
  v.store = STORE_D;
  v.out = M;
  v.map_stride_out = B;
  v.op[0] = OP_COS; v.op[1] = OP_SIN; v.op[2] = OP_COS; v.op[3] = OP_COS;
  if ((rc = run_pass(v, 0, g, 4, s))) return rc;
  v.load = LOAD_D;
  v.in = M;
  v.map_stride_in = B;
  v.in_scale = 1.0;
  v.op[0] = OP_COS; v.op[1] = OP_COS; v.op[2] = OP_SIN; v.op[3] = OP_COS;
  if ((rc = run_pass(v, 1, g, 4, s))) return rc;
  v.store = STORE_MAPS;
  v.out = maps;
  v.op[0] = OP_COS; v.op[1] = OP_COS; v.op[2] = OP_COS; v.op[3] = OP_SIN;
  if ((rc = run_pass(v, 2, g, 4, s))) return rc;
  return P3D_OK;
}

}  // namespace p3d
