// Small per-op entry points of the reference's Python operator API that the
// fused loop computes inline (so they exist as kernels for callers that use
// the ops one by one): dynamic_size (density.py:134-147), the 3-D prefix /
// suffix sums of the macro corner maps (density.py:207-217), overflow of a
// float64 map (density.py:612-617), NetBoxes.spans (wirelength.py:136-142)
// and the two reductions plus the update of NesterovOptimizer.advance
// (gp.py:203-226).  Compiled with -fmad=false: numpy's rounding.
#include <math.h>

#include "p3d_common.cuh"
#include "p3d_geom.cuh"
#include "p3d_internal.cuh"

namespace p3d {

namespace {

__global__ void dynamic_size_kernel(int n, const double* wt, const double* ht, const double* wb,
                                    const double* hb, const uint8_t* mac, const double* z,
                                    double dz, double* w, double* h) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    dynamic_wh(z[i], dz, mac[i] != 0, wt[i], ht[i], wb[i], hb[i], w[i], h[i]);
}

// inclusive scan along one axis of a C-ordered [nx][ny][nz] map, one thread
// per line (sequential adds in index order: numpy's cumsum order)
__global__ void axis_scan_kernel(int nx, int ny, int nz, int axis, bool reverse, double* a) {
  const long long lines = axis == 0 ? (long long)ny * nz : (axis == 1 ? (long long)nx * nz : (long long)nx * ny);
  const int len = axis == 0 ? nx : (axis == 1 ? ny : nz);
  const long long stride = axis == 0 ? (long long)ny * nz : (axis == 1 ? nz : 1);
  for (long long l = blockIdx.x * (long long)blockDim.x + threadIdx.x; l < lines;
       l += (long long)gridDim.x * blockDim.x) {
    long long base;
    if (axis == 0) base = l;                                   // (j, k)
    else if (axis == 1) base = (l / nz) * ny * nz + (l % nz);  // (i, k)
    else base = l * nz;                                        // (i, j)
    double s = 0.0;
    for (int t = 0; t < len; ++t) {
      const long long p = base + (long long)(reverse ? len - 1 - t : t) * stride;
      s += a[p];
      a[p] = s;
    }
  }
}

__global__ void overflow_d_kernel(long long n, const double* rho, double rho_t, double scale,
                                  double* partials, unsigned int* counter, double* out) {
  __shared__ double red[32];
  double acc[1] = {0.0};
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const double e = rho[i] - rho_t;
    acc[0] += e > 0.0 ? e : 0.0;
  }
  block_sum<1>(acc, red);
  if (threadIdx.x == 0) partials[blockIdx.x] = acc[0];
  if (last_block(counter)) {
    const double s = ordered_sum(partials, gridDim.x, red);
    if (threadIdx.x == 0) *out = s * scale;
  }
}

__global__ void spans_kernel(int n, const int64_t* cnt, const double* min1, const double* max1,
                             const double* fmin, const double* fmax, double* top, double* bot,
                             double* full) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
    const long long c0 = cnt[2 * j], c1 = cnt[2 * j + 1];
    top[j] = c1 > 0 ? max1[2 * j + 1] - min1[2 * j + 1] : 0.0;
    bot[j] = c0 > 0 ? max1[2 * j] - min1[2 * j] : 0.0;
    full[j] = (c0 + c1) > 0 ? fmax[j] - fmin[j] : 0.0;
  }
}

// |v - v_prev|^2 and |g - ref|^2 (the BB numerator / denominator, gp.py:210-212)
__global__ void bb_norms_kernel(long long n, const double* v, const double* vp, const double* g,
                                const double* ref, double* partials, unsigned int* counter,
                                double* out) {
  __shared__ double red[64];
  double acc[2] = {0.0, 0.0};
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const double a = v[i] - vp[i], b = g[i] - ref[i];
    acc[0] += a * a;
    acc[1] += b * b;
  }
  block_sum<2>(acc, red);
  if (threadIdx.x == 0) {
    partials[blockIdx.x] = acc[0];
    partials[kMaxBlocks + blockIdx.x] = acc[1];
  }
  if (last_block(counter)) {
    const double a = ordered_sum(partials, gridDim.x, red);
    const double b = ordered_sum(partials + kMaxBlocks, gridDim.x, red);
    if (threadIdx.x == 0) { out[0] = a; out[1] = b; out[2] = 0.0; }
  }
}

__global__ void absmax_kernel(long long n, const double* g, double* partials,
                              unsigned int* counter, double* out) {
  __shared__ double red[32];
  double m = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    m = fmax(m, fabs(g[i]));
  m = block_max(m, red);
  if (threadIdx.x == 0) partials[blockIdx.x] = m;
  if (last_block(counter)) {
    const double v = block_max_partials((volatile double*)partials, gridDim.x, red);
    if (threadIdx.x == 0) *out = v;
  }
}

// out = a + s * (b - c)   (c nullable: out = a + s * b)
__global__ void axpy_kernel(long long n, const double* a, double s, const double* b,
                            const double* c, double* out) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    out[i] = a[i] + s * (c ? b[i] - c[i] : b[i]);
}

}  // namespace

void launch_dynamic_size(int n, const double* wt, const double* ht, const double* wb,
                         const double* hb, const uint8_t* mac, const double* z, double dz,
                         double* w, double* h, cudaStream_t s) {
  dynamic_size_kernel<<<grid_blocks(n, 256, kMaxBlocks), 256, 0, s>>>(n, wt, ht, wb, hb, mac, z, dz, w, h);
}
void launch_axis_scan(int nx, int ny, int nz, int axis, bool reverse, double* a, cudaStream_t s) {
  const long long lines = axis == 0 ? (long long)ny * nz : (axis == 1 ? (long long)nx * nz : (long long)nx * ny);
  axis_scan_kernel<<<grid_blocks((int)(lines < 0x7fffffffLL ? lines : 0x7fffffffLL), 128, kMaxBlocks), 128, 0, s>>>(nx, ny, nz, axis, reverse, a);
}
void launch_overflow_d(long long n, const double* rho, double rho_t, double scale, double* scratch,
                       double* out, cudaStream_t s) {
  overflow_d_kernel<<<grid_blocks((int)(n < 0x7fffffffLL ? n : 0x7fffffffLL), 256, 1024), 256, 0, s>>>(
      n, rho, rho_t, scale, scratch + 8, reinterpret_cast<unsigned int*>(scratch), out);
}
void launch_spans(int n, const int64_t* cnt, const double* min1, const double* max1,
                  const double* fmin, const double* fmax, double* top, double* bot, double* full,
                  cudaStream_t s) {
  spans_kernel<<<grid_blocks(n, 256, kMaxBlocks), 256, 0, s>>>(n, cnt, min1, max1, fmin, fmax, top, bot, full);
}
void launch_bb_norms(long long n, const double* v, const double* vp, const double* g,
                     const double* ref, double* scratch, double* out, cudaStream_t s) {
  bb_norms_kernel<<<grid_blocks((int)(n < 0x7fffffffLL ? n : 0x7fffffffLL), 256, 1024), 256, 0, s>>>(
      n, v, vp, g, ref, scratch + 8, reinterpret_cast<unsigned int*>(scratch), out);
}
void launch_absmax(long long n, const double* g, double* scratch, double* out, cudaStream_t s) {
  absmax_kernel<<<grid_blocks((int)(n < 0x7fffffffLL ? n : 0x7fffffffLL), 256, 1024), 256, 0, s>>>(
      n, g, scratch + 8, reinterpret_cast<unsigned int*>(scratch), out);
}
void launch_axpy(long long n, const double* a, double sc, const double* b, const double* c,
                 double* out, cudaStream_t s) {
  axpy_kernel<<<grid_blocks((int)(n < 0x7fffffffLL ? n : 0x7fffffffLL), 256, kMaxBlocks), 256, 0, s>>>(n, a, sc, b, c, out);
}

}  // namespace p3d
