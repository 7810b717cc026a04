// K2 / K4 per-op entry kernels and small per-object ops.  Compiled with
// -fmad=false: the overlap arithmetic must be bit-identical to numpy's.
//
// K2  accumulate_density (density.py:301-311): cells and fillers scatter their
//     (object, bin) overlaps thread-per-object; macros take one CTA each and
//     scatter their whole footprint tile (per-macro tile path).  Terms are
//     quantised to int64 (2^-40 per unit density) and added with integer
//     atomics, so the map is exact and independent of execution order.
// K4  density_energy / density_force (density.py:568-609): thread-per-object
//     overlap-weighted means of the interleaved (phi, Ex, Ey, Ez) map, one CTA
//     per macro.
#include "p3d_geom.cuh"
#include "p3d_internal.cuh"

namespace p3d {

template <class Cloud>
__global__ void __launch_bounds__(256) scatter_cells_kernel(Cloud cl, int n, p3d_grid g,
                                                           unsigned long long* rho,
                                                           const int* halt) {
  if (halt && *halt) return;
  const int stride = gridDim.x * blockDim.x;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    if (cl.is_macro(i)) continue;
    scatter_object(cl.get(i), g, rho);
  }
}

template <class Cloud>
__global__ void __launch_bounds__(256) scatter_macros_kernel(Cloud cl, const int32_t* ids,
                                                            p3d_grid g, unsigned long long* rho,
                                                            const int* halt) {
  if (halt && *halt) return;
  scatter_object_block(cl.get(ids[blockIdx.x]), g, rho);
}

template <class Cloud>
void launch_scatter(const Cloud& cl, int n, int n_macro, const int32_t* macro_ids,
                    const p3d_grid& g, int64_t* rho, const int* halt, cudaStream_t s) {
  unsigned long long* r = reinterpret_cast<unsigned long long*>(rho);
  if (n > 0) scatter_cells_kernel<<<grid_blocks(n, 256, 148 * 16), 256, 0, s>>>(cl, n, g, r, halt);
  if (n_macro > 0) scatter_macros_kernel<<<n_macro, 256, 0, s>>>(cl, macro_ids, g, r, halt);
}

template void launch_scatter<CloudGP>(const CloudGP&, int, int, const int32_t*, const p3d_grid&,
                                      int64_t*, const int*, cudaStream_t);
template void launch_scatter<CloudArrays>(const CloudArrays&, int, int, const int32_t*,
                                          const p3d_grid&, int64_t*, const int*, cudaStream_t);

// ---------------------------------------------------------------------------
// per-op density gather: energy = sum q*phibar, force = -2 q Ebar
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) gather_op_kernel(CloudArrays cl, p3d_grid g,
                                                       const double* maps,
                                                       const uint8_t* freeze, double* force,
                                                       double* partials, unsigned int* counter,
                                                       double* energy) {
  __shared__ double red[32 * 4];
  double e[1] = {0.0};
  const int n = cl.c.n;
  const int nm = cl.c.n_macro;
  if ((int)blockIdx.x < nm) {  // one CTA per macro
    const int i = cl.c.macro_ids[blockIdx.x];
    const Charge q = cl.get(i);
    double mean[4];
    gather_object_block(q, g, maps, mean, red);
    if (threadIdx.x == 0) {
      const double qq = charge_of(q);
      const double c = -2.0 * qq;
      force[3 * i + 0] = mean[1] * c;
      force[3 * i + 1] = mean[2] * c;
      force[3 * i + 2] = (freeze && freeze[i]) ? 0.0 : mean[3] * c;
      e[0] = qq * mean[0];
    }
  } else {
    const int b = blockIdx.x - nm, nb = gridDim.x - nm;
    for (int i = b * blockDim.x + threadIdx.x; i < n; i += nb * blockDim.x) {
      if (cl.is_macro(i)) continue;
      const Charge q = cl.get(i);
      double mean[4];
      gather_object(q, g, maps, mean);
      const double qq = charge_of(q);
      const double c = -2.0 * qq;
      force[3 * i + 0] = mean[1] * c;
      force[3 * i + 1] = mean[2] * c;
      force[3 * i + 2] = (freeze && freeze[i]) ? 0.0 : mean[3] * c;
      e[0] += qq * mean[0];
    }
  }
  block_sum<1>(e, red);
  if (threadIdx.x == 0) partials[blockIdx.x] = e[0];
  if (last_block(counter)) {
    double s = ordered_sum(partials, gridDim.x, red);
    if (threadIdx.x == 0) *energy = s;
  }
}

void launch_gather_op(const p3d_cloud& c, const p3d_grid& g, const double* maps,
                      const uint8_t* freeze, double* energy, double* force, double* scratch,
                      cudaStream_t s) {
  CloudArrays cl;
  cl.c = c;
  const int nb = grid_blocks(c.n, 256, 1024);
  unsigned int* counter = reinterpret_cast<unsigned int*>(scratch);
  double* partials = scratch + 8;
  gather_op_kernel<<<c.n_macro + nb, 256, 0, s>>>(cl, g, maps, freeze, force, partials, counter,
                                                 energy);
}

// ---------------------------------------------------------------------------
// small elementwise / reduction ops of the per-op API
// ---------------------------------------------------------------------------
__global__ void fx_to_density_kernel(long long n, const int64_t* in, double* out) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    out[i] = (double)in[i] * 9.094947017729282379150390625e-13;  // 2^-40
}

void launch_fx_to_density(long long n, const int64_t* in, double* out, cudaStream_t s) {
  int b = (int)((n + 255) / 256);
  b = b < 1 ? 1 : (b > 4096 ? 4096 : b);
  fx_to_density_kernel<<<b, 256, 0, s>>>(n, in, out);
}

__global__ void overflow_kernel(long long n, const int64_t* rho, long long t, double scale,
                                long long* partials, unsigned int* counter, double* out) {
  long long e = 0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    long long d = rho[i] - t;
    e += d > 0 ? d : 0;
  }
  e = warp_sum_ll(e);
  __shared__ long long ws[32];
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = e;
  __syncthreads();
  if (threadIdx.x == 0) {
    long long b = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) b += ws[w];
    partials[blockIdx.x] = b;
  }
  if (last_block(counter)) {
    if (threadIdx.x == 0) {
      long long s = 0;
      for (int i = 0; i < (int)gridDim.x; ++i) s += ((volatile long long*)partials)[i];
      *out = (double)s * scale;
    }
  }
}

void launch_overflow(long long n, const int64_t* rho, long long t, double scale, double* scratch,
                     double* out, cudaStream_t s) {
  int b = (int)((n + 255) / 256);
  b = b < 1 ? 1 : (b > 1024 ? 1024 : b);
  overflow_kernel<<<b, 256, 0, s>>>(n, rho, t, scale, reinterpret_cast<long long*>(scratch + 8),
                                    reinterpret_cast<unsigned int*>(scratch), out);
}

// gp.py:142-147
__global__ void precondition_kernel(int n, const double* g, double lam, const double* q,
                                    const double* deg, const uint8_t* macro, double* out,
                                    double* div) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    double d = lam * q[i];
    d = d + ((macro && macro[i]) ? deg[i] : 0.0);
    d = fmax(d, 1.0);
    if (div) div[i] = d;
    out[3 * i + 0] = g[3 * i + 0] / d;
    out[3 * i + 1] = g[3 * i + 1] / d;
    out[3 * i + 2] = g[3 * i + 2] / d;
  }
}

void launch_precondition(int n, const double* g, double lam, const double* q, const double* deg,
                         const uint8_t* macro, double* out, double* div, cudaStream_t s) {
  precondition_kernel<<<grid_blocks(n, 256, 4096), 256, 0, s>>>(n, g, lam, q, deg, macro, out, div);
}

// wirelength.py:308-322
__global__ void pin_coords_kernel(int n_pin, const int32_t* pin_inst, const double* x,
                                  const double* y, const double* z, const double* off, double dz,
                                  double* px, double* py, double* pz, uint8_t* top) {
  const double dz2 = dz / 2;
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n_pin; k += gridDim.x * blockDim.x) {
    const int i = pin_inst[k];
    const double zi = z[i];
    const bool t = (zi - dz2) > 0.0;
    const double* o = off + 4 * (long long)k;
    if (px) px[k] = x[i] + (t ? o[0] : o[2]);
    if (py) py[k] = y[i] + (t ? o[1] : o[3]);
    if (pz) pz[k] = zi;
    if (top) top[k] = t;
  }
}

void launch_pin_coords(int n_pin, const int32_t* pin_inst, const double* x, const double* y,
                       const double* z, const double* off, double dz, double* px, double* py,
                       double* pz, uint8_t* top, cudaStream_t s) {
  pin_coords_kernel<<<grid_blocks(n_pin, 256, 4096), 256, 0, s>>>(n_pin, pin_inst, x, y, z, off,
                                                                 dz, px, py, pz, top);
}

// wirelength.py:296-305: two-phase (deterministic) L1 norms then the combine
__global__ void l1_kernel(int n, const double* gx, const double* gy, const double* gzb,
                          double* partials, unsigned int* counter, double* norms) {
  __shared__ double red[32 * 3];
  double acc[3] = {0, 0, 0};
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    acc[0] += fabs(gx[i]);
    acc[1] += fabs(gy[i]);
    acc[2] += fabs(gzb[i]);
  }
  block_sum<3>(acc, red);
  if (threadIdx.x == 0)
    for (int q = 0; q < 3; ++q) partials[q * gridDim.x + blockIdx.x] = acc[q];
  if (last_block(counter)) {
    for (int q = 0; q < 3; ++q) {
      double s = ordered_sum(partials + q * gridDim.x, gridDim.x, red);
      if (threadIdx.x == 0) norms[q] = s;
    }
  }
}

__global__ void normalize_kernel(int n, const double* gzb, const double* gzh, double alpha,
                                 const double* norms, double* out) {
  const double nz = norms[2];
  const double scale = nz == 0.0 ? 0.0 : (norms[0] + norms[1]) / (2 * nz);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const double base = nz == 0.0 ? 0.0 : scale * gzb[i];
    out[i] = base + alpha * gzh[i];
  }
}

void launch_normalize(int n, const double* gx, const double* gy, const double* gzb,
                      const double* gzh, double alpha, double* out, double* scratch,
                      cudaStream_t s) {
  const int b = grid_blocks(n, 256, 1024);
  unsigned int* counter = reinterpret_cast<unsigned int*>(scratch);
  double* norms = scratch + 4;
  double* partials = scratch + 8;
  l1_kernel<<<b, 256, 0, s>>>(n, gx, gy, gzb, partials, counter, norms);
  normalize_kernel<<<grid_blocks(n, 256, 4096), 256, 0, s>>>(n, gzb, gzh, alpha, norms, out);
}

}  // namespace p3d
