// Shared device helpers and the parameter blocks of the GP hot path.
// See DESIGN.md for the HBM layout and include/p3d.h for the C-ABI.
#pragma once

#include <stdlib.h>

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/p3d.h"

#define P3D_INF (__longlong_as_double(0x7ff0000000000000LL))

namespace p3d {

// one-time per-device setup (function attributes, side streams) is keyed by
// the current device: cudaFuncSetAttribute and streams are per context
constexpr int kMaxDevices = 64;
inline int current_device() {
  int d = 0;
  cudaGetDevice(&d);
  return d < 0 ? 0 : (d >= kMaxDevices ? kMaxDevices - 1 : d);
}

constexpr int kFxBits = 40;  // fixed-point density: 2^-40 per unit density

// ---------------------------------------------------------------------------
// error reporting (host)
// ---------------------------------------------------------------------------
void set_error(const char* fmt, ...);
int check_launch(const char* what);

// ---------------------------------------------------------------------------
// programmatic dependent launch (PDL): the loop's kernels are launched with
// programmatic stream serialisation so a kernel's launch overlaps its
// predecessor's tail; every such kernel waits for the predecessor's memory
// (griddepcontrol.wait) before its first global access, so the semantics are
// those of plain stream order.  A no-op when launched without the attribute.
// ---------------------------------------------------------------------------
#ifndef P3D_PDL
#define P3D_PDL 1
#endif
__device__ __forceinline__ void pdl_wait() {
#if P3D_PDL
  asm volatile("griddepcontrol.wait;" ::: "memory");
#endif
}

// P3D_NOPDL (environment, A/B only): bitmask of launch groups started without
// the PDL attribute (1 K1 net, 2 K1b gather, 4 K2, 8 K3, 16 K4, 32 K5a, 64 K5b)
inline int nopdl_mask() {
  static const int m = getenv("P3D_NOPDL") ? atoi(getenv("P3D_NOPDL")) : 0;
  return m;
}
template <typename... KArgs, typename... Args>
inline cudaError_t pdl_launch_tag(int tag, void (*kernel)(KArgs...), dim3 grid, dim3 block,
                                  size_t smem, cudaStream_t s, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = P3D_PDL && !(nopdl_mask() & tag);
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

template <typename... KArgs, typename... Args>
inline cudaError_t pdl_launch(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                              cudaStream_t s, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = P3D_PDL;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

// Store a double with an L2 evict-last policy (data the next kernel gathers
// from: field maps, the step's pos4 copy).  -DP3D_L2_KEEP=0 disables.
#ifndef P3D_L2_KEEP
#define P3D_L2_KEEP 1
#endif
__device__ __forceinline__ void st_keep(double* p, double v) {
#if P3D_L2_KEEP
  unsigned long long pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(p), "d"(v), "l"(pol) : "memory");
#else
  *p = v;
#endif
}
__device__ __forceinline__ void st_keep2(double* p, double a, double b) {  // 16-byte aligned
#if P3D_L2_KEEP
  unsigned long long pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;" ::"l"(p), "d"(a), "d"(b),
               "l"(pol)
               : "memory");
#else
  p[0] = a;
  p[1] = b;
#endif
}

// ---------------------------------------------------------------------------
// warp / block reductions (deterministic: fixed shuffle tree, fixed order)
// ---------------------------------------------------------------------------
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ long long warp_sum_ll(long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Block-wide sum of K doubles per thread; result valid in thread 0.
// blockDim.x must be a multiple of 32 and <= 1024.
template <int K>
__device__ __forceinline__ void block_sum(double (&v)[K], double* smem /* >= 32*K */) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int k = 0; k < K; ++k) v[k] = warp_sum(v[k]);
  __syncthreads();
  if (lane == 0) {
#pragma unroll
    for (int k = 0; k < K; ++k) smem[k * 32 + wid] = v[k];
  }
  __syncthreads();
  if (wid == 0) {
#pragma unroll
    for (int k = 0; k < K; ++k) {
      double t = lane < nw ? smem[k * 32 + lane] : 0.0;
      v[k] = warp_sum(t);
    }
  }
  __syncthreads();
}

__device__ __forceinline__ double block_max(double v, double* smem) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  v = warp_max(v);
  __syncthreads();
  if (lane == 0) smem[wid] = v;
  __syncthreads();
  if (wid == 0) {
    double t = lane < nw ? smem[lane] : 0.0;
    v = warp_max(t);
  }
  __syncthreads();
  return v;
}

// "Last block done" handshake: every block publishes its partials (written by
// thread 0, after the block reduction), then the last block to arrive (by an
// atomic ticket) sees all of them and runs the grid-level epilogue.  Only
// thread 0 fences (it wrote the partials), so the other warps of a block do
// not wait for their own outstanding stores.  The ticket counter resets itself
// for graph replay.
__device__ __forceinline__ bool last_block(unsigned int* counter) {
  __shared__ bool is_last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    unsigned int t = atomicAdd(counter, 1u);
    is_last = (t == gridDim.x * gridDim.y - 1);
    if (is_last) *counter = 0u;
  }
  __syncthreads();
  if (is_last) __threadfence();
  return is_last;
}

// last_block for kernels whose every thread published global data (e.g.
// atomics) the last block must see: all threads fence before the ticket.
__device__ __forceinline__ bool last_block_all(unsigned int* counter) {
  __threadfence();
  return last_block(counter);
}

// Ordered sum of n partials by one block (fixed order => deterministic).
__device__ __forceinline__ double ordered_sum(const volatile double* p, int n, double* smem) {
  double acc[1] = {0.0};
  // contiguous chunk per thread, then fixed tree
  int per = (n + blockDim.x - 1) / blockDim.x;
  int b = threadIdx.x * per, e = min(n, b + per);
  double s = 0.0;
  for (int i = b; i < e; ++i) s += p[i];
  acc[0] = s;
  block_sum<1>(acc, smem);
  return acc[0];  // valid in thread 0
}

// K ordered sums at once (partials of sum k at p + k * stride): the same
// per-thread chunks and the same tree as K calls of ordered_sum, so the
// results are identical, but every partial load is in flight together and
// the block reduces once (the last-block tails of the loop kernels).
template <int K>
__device__ __forceinline__ void ordered_sums(const volatile double* p, int stride, int n,
                                             double* smem /* >= 32*K */, double (&out)[K]) {
  const int per = (n + blockDim.x - 1) / blockDim.x;
  const int b = threadIdx.x * per, e = min(n, b + per);
#pragma unroll
  for (int k = 0; k < K; ++k) out[k] = 0.0;
  for (int i = b; i < e; ++i) {
#pragma unroll
    for (int k = 0; k < K; ++k) out[k] += p[k * stride + i];
  }
  block_sum<K>(out, smem);  // valid in thread 0
}

// Sum of n int64 partials by the whole block (integer: order-independent);
// result valid in thread 0.
__device__ __forceinline__ long long block_sum_ll_partials(const volatile long long* p, int n) {
  __shared__ long long ws[32];
  long long s = 0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) s += p[i];
  s = warp_sum_ll(s);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = s;
  __syncthreads();
  long long t = 0;
  if (threadIdx.x == 0)
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += ws[w];
  return t;
}

// Max of n double partials by the whole block; result valid in thread 0.
__device__ __forceinline__ double block_max_partials(const volatile double* p, int n, double* smem) {
  double m = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) m = fmax(m, p[i]);
  return block_max(m, smem);
}

// ---------------------------------------------------------------------------
// numpy-faithful small math (compiled with -fmad=false where used)
// ---------------------------------------------------------------------------
// max / min of two doubles as one compare and a select (fmax / fmin spend ~7
// SASS instructions on NaN handling).  Identical to fmax / fmin whenever
// neither argument is NaN; every caller passes finite coordinates / spans
// (or +-inf sentinels).
__device__ __forceinline__ double dmax(double a, double b) { return a > b ? a : b; }
__device__ __forceinline__ double dmin(double a, double b) { return a < b ? a : b; }

// x / b from y = 1/b (one IEEE division shared by several quotients with the
// same divisor): q = x y, then one exact FMA residual correction.  With
// y = RN(1/b) this is Markstein's correctly rounded quotient, i.e. the same
// value as the IEEE division, for results in the normal range (every caller:
// preconditioner divisors >= 1, overlap volumes >= 1e-300 with numerators
// bounded by them); -DP3D_SHARED_RCP=0 restores plain divisions.
#ifndef P3D_SHARED_RCP
#define P3D_SHARED_RCP 1
#endif
__device__ __forceinline__ double div_rcp(double x, double b, double y) {
#if P3D_SHARED_RCP
  const double q = x * y;
  return fma(fma(-q, b, x), y, q);
#else
  return x / b;
#endif
}

__device__ __forceinline__ double clipd(double v, double lo, double hi) {
  // np.clip(v, lo, hi) == minimum(maximum(v, lo), hi) for lo <= hi (every
  // caller); a NaN v stays NaN as in numpy
  return v < lo ? lo : (v > hi ? hi : v);
}

}  // namespace p3d
