// Post-GP steps of the reference flow: the die
// utilisation rebalance (legalize.py:464-499 rebalance_partition) and the
// independent solution check (check.py:74-152 check_solution).
//
// rebalance: the reference moves, one instance per step, the cheapest
// instance (cells before macros, then smallest area on its die, then index)
// off the die whose utilisation overshoots more, recomputing both dies' areas
// each step, until both caps hold (or both are exceeded: unsatisfiable).  A
// step changes nothing but the moved instance, so between two changes of the
// source die the moves are a prefix of the source die's sorted candidate
// list: one CTA walks that list (pre-sorted on the device per die) in chunks,
// with block prefix sums of the two dies' areas giving the state before every
// candidate move, and stops at the first candidate whose preceding state ends
// the phase (caps met, both exceeded, or the other die now overshoots more).
// Area sums are float64 running sums; they are exact (so every decision equals
// the reference's) whenever the instance areas are integers below 2^53 (the
// synthetic and database-unit designs).
//
// check: per-instance rotation / bounds / row / site flags and per-die area;
// per-net crossing vs terminal flags; terminal bounds; and the two pair
// searches (same-die instance overlaps, terminal spacing) by a uniform bucket
// grid (the reference's spatial hash, check.py:47-71): every box is entered in
// all buckets it touches, each bucket tests its pairs, and a pair is reported
// only by the bucket holding the lower-left corner of the two boxes'
// intersection (so once).  The host formats the messages of the flagged
// items from the caller's own solution objects.
#include <math.h>

#include "p3d_common.cuh"
#include "p3d_internal.cuh"

namespace p3d {

namespace {

constexpr int kRbThreads = 1024;

// inclusive block scan of (a, b, c) over 1024 threads; returns exclusive
// prefixes and the block totals
__device__ __forceinline__ void block_scan3(double a, double b, int c, double& ea, double& eb,
                                            int& ec, double& ta, double& tb, int& tc) {
  __shared__ double sa[32], sb[32];
  __shared__ int sc[32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  double xa = a, xb = b;
  int xc = c;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double ya = __shfl_up_sync(0xffffffffu, xa, o);
    const double yb = __shfl_up_sync(0xffffffffu, xb, o);
    const int yc = __shfl_up_sync(0xffffffffu, xc, o);
    if (lane >= o) { xa += ya; xb += yb; xc += yc; }
  }
  __syncthreads();
  if (lane == 31) { sa[wid] = xa; sb[wid] = xb; sc[wid] = xc; }
  __syncthreads();
  if (wid == 0) {
    double wa = lane < nw ? sa[lane] : 0.0, wb = lane < nw ? sb[lane] : 0.0;
    int wc = lane < nw ? sc[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const double ya = __shfl_up_sync(0xffffffffu, wa, o);
      const double yb = __shfl_up_sync(0xffffffffu, wb, o);
      const int yc = __shfl_up_sync(0xffffffffu, wc, o);
      if (lane >= o) { wa += ya; wb += yb; wc += yc; }
    }
    sa[lane] = wa; sb[lane] = wb; sc[lane] = wc;
  }
  __syncthreads();
  const double pa = wid ? sa[wid - 1] : 0.0, pb = wid ? sb[wid - 1] : 0.0;
  const int pc = wid ? sc[wid - 1] : 0;
  ea = pa + xa - a;
  eb = pb + xb - b;
  ec = pc + xc - c;
  ta = sa[nw - 1];
  tb = sb[nw - 1];
  tc = sc[nw - 1];
  __syncthreads();
}

__global__ void __launch_bounds__(kRbThreads) rebalance_kernel(RebalanceArgs a) {
  __shared__ double red[32 * 2];
  __shared__ int first;
  const int n = a.n;
  // initial areas (legalize.py:479-480), per-thread contiguous chunks
  double acc[2] = {0.0, 0.0};
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    if (a.delta[i] & 1) acc[0] += a.area_top[i];
    else acc[1] += a.area_bot[i];
  }
  block_sum<2>(acc, red);
  __shared__ double At_s, Ab_s;
  if (threadIdx.x == 0) { At_s = acc[0]; Ab_s = acc[1]; }
  __syncthreads();
  double At = At_s, Ab = Ab_s;
  long long moves = 0;
  const double capT = a.cap_top, capB = a.cap_bot;
  int status = 2;  // did not converge
  bool exhausted_prev = false;
  int src_prev = -1;
  while (true) {
    if (moves >= (long long)n + 1) { status = 2; break; }
    if (At <= capT && Ab <= capB) { status = 0; break; }
    const double oT = At - capT, oB = Ab - capB;
    if (oT > 0 && oB > 0) { status = 1; break; }
    const int src = oT >= oB ? 1 : 0;
    if (exhausted_prev && src == src_prev) { status = 2; break; }  // no candidate left
    const int* ord = src ? a.order_top : a.order_bot;
    const double* as_ = src ? a.area_top : a.area_bot;
    const double* ao_ = src ? a.area_bot : a.area_top;
    bool ended = false;
    for (int base = 0; base < n && !ended; base += blockDim.x) {
      const int p = base + threadIdx.x;
      const int i = p < n ? ord[p] : -1;
      const bool valid = i >= 0 && (a.delta[i] & 1) == src;
      const double vs = valid ? as_[i] : 0.0, vo = valid ? ao_[i] : 0.0;
      double es, eo, ts, to;
      int ec, tc;
      block_scan3(vs, vo, valid ? 1 : 0, es, eo, ec, ts, to, tc);
      // the state before this candidate's move
      bool event = false;
      if (valid) {
        const double at = src ? At - es : At + eo, ab = src ? Ab + eo : Ab - es;
        const double ot = at - capT, ob = ab - capB;
        event = (at <= capT && ab <= capB) || (ot > 0 && ob > 0) || ((ot >= ob ? 1 : 0) != src) ||
                (moves + ec >= (long long)n + 1);
      }
      if (threadIdx.x == 0) first = 0x7fffffff;
      __syncthreads();
      if (event) atomicMin(&first, p);
      __syncthreads();
      const int f = first;
      if (f != 0x7fffffff) {
        // moves before f only: totals of the valid candidates before it
        const bool mv = valid && p < f;
        double e2s, e2o, t2s, t2o;
        int e2c, t2c;
        block_scan3(mv ? vs : 0.0, mv ? vo : 0.0, mv ? 1 : 0, e2s, e2o, e2c, t2s, t2o, t2c);
        if (mv) a.delta[i] = (uint8_t)((1 - src) | 2);
        ts = t2s; to = t2o; tc = t2c;
        ended = true;
      } else if (valid) {
        a.delta[i] = (uint8_t)((1 - src) | 2);
      }
      if (src) { At -= ts; Ab += to; } else { Ab -= ts; At += to; }
      moves += tc;
      __syncthreads();
    }
    exhausted_prev = !ended;
    src_prev = src;
  }
  if (threadIdx.x == 0) {
    a.out[0] = status;
    a.out[1] = (double)moves;
    a.out[2] = At - capT;
    a.out[3] = Ab - capB;
  }
}

// ---- check_solution ------------------------------------------------------
// per instance: bit 0 rotated cell, 1 bounds, 2 row, 3 site (check.py:78-101)
__global__ void check_inst_kernel(CheckArgs a) {
  __shared__ double red[32 * 2];
  double area[2] = {0.0, 0.0};
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < a.n_inst; i += gridDim.x * blockDim.x) {
    const int d = a.die[i];
    const int q = ((a.rot[i] % 4) + 4) % 4;
    const bool mac = a.is_macro[i] != 0;
    const double kw = d ? a.w_top[i] : a.w_bot[i], kh = d ? a.h_top[i] : a.h_bot[i];
    const double w = (q & 1) ? kh : kw, h = (q & 1) ? kw : kh;
    const double x0 = a.x[i], y0 = a.y[i];
    int f = 0;
    if (!mac && q != 0) f |= 1;
    if (x0 < -a.tol || y0 < -a.tol || x0 + w > a.die_w + a.tol || y0 + h > a.die_h + a.tol) f |= 2;
    if (!mac) {
      const double rh = d ? a.row_top : a.row_bot;
      const double r = y0 / rh;
      if (fabs(r - rint(r)) > a.tol) f |= 4;
      const double s = x0 / a.site_w;
      if (fabs(s - rint(s)) > a.tol) f |= 8;
    }
    a.inst_flags[i] = (uint8_t)f;
    a.box[4 * (long long)i + 0] = x0;
    a.box[4 * (long long)i + 1] = x0 + w;
    a.box[4 * (long long)i + 2] = y0;
    a.box[4 * (long long)i + 3] = y0 + h;
    area[d ? 1 : 0] += w * h;
  }
  block_sum<2>(area, red);
  if (threadIdx.x == 0) {
    a.partials[blockIdx.x] = area[0];
    a.partials[kMaxBlocks + blockIdx.x] = area[1];
  }
  if (last_block(a.counter)) {
    const double a0 = ordered_sum(a.partials, gridDim.x, red);
    const double a1 = ordered_sum(a.partials + kMaxBlocks, gridDim.x, red);
    if (threadIdx.x == 0) { a.area[0] = a0; a.area[1] = a1; }
  }
}

// per net: bit 0 crossing without terminal, bit 1 single-die with one
// (check.py:117-124); per terminal: bit 2 out of bounds (check.py:127-129)
__global__ void check_net_kernel(CheckArgs a) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < a.n_net; j += gridDim.x * blockDim.x) {
    int mn = 2, mx = -1;
    for (int k = a.net_ptr[j]; k < a.net_ptr[j + 1]; ++k) {
      const int d = a.die[a.pin_inst[k]] ? 1 : 0;
      mn = min(mn, d);
      mx = max(mx, d);
    }
    const bool crossing = mx > mn;
    const bool has = a.hbt_ok[j] != 0;
    int f = 0;
    if (crossing && !has) f |= 1;
    if (!crossing && has) f |= 2;
    if (has) {
      const double hx = a.hbt_x[j], hy = a.hbt_y[j];
      if (hx < -a.tol || hy < -a.tol || hx + a.pitch > a.die_w + a.tol || hy + a.pitch > a.die_h + a.tol)
        f |= 4;
    }
    a.net_flags[j] = (uint8_t)f;
  }
}

// ---- bucket-grid pair search -------------------------------------------
__device__ __forceinline__ int bucket_of(double v, double bucket, int nb) {
  const double q = floor(v / bucket);
  return q < 0 ? 0 : (q >= nb ? nb - 1 : (int)q);
}

__global__ void pair_count_kernel(PairArgs a) {
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < a.n; k += gridDim.x * blockDim.x) {
    if (!a.member[k]) continue;
    const double* b = a.box + 4 * (long long)k;
    const int i0 = bucket_of(b[0], a.bucket, a.nbx), i1 = bucket_of(b[1], a.bucket, a.nbx);
    const int j0 = bucket_of(b[2], a.bucket, a.nby), j1 = bucket_of(b[3], a.bucket, a.nby);
    for (int i = i0; i <= i1; ++i)
      for (int j = j0; j <= j1; ++j) atomicAdd(&a.count[i * a.nby + j], 1);
  }
}

__global__ void pair_fill_kernel(PairArgs a) {
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < a.n; k += gridDim.x * blockDim.x) {
    if (!a.member[k]) continue;
    const double* b = a.box + 4 * (long long)k;
    const int i0 = bucket_of(b[0], a.bucket, a.nbx), i1 = bucket_of(b[1], a.bucket, a.nbx);
    const int j0 = bucket_of(b[2], a.bucket, a.nby), j1 = bucket_of(b[3], a.bucket, a.nby);
    for (int i = i0; i <= i1; ++i)
      for (int j = j0; j <= j1; ++j) a.list[atomicAdd(&a.cursor[i * a.nby + j], 1)] = k;
  }
}

// one CTA per bucket: every pair (a < c by object index) of the bucket
__global__ void pair_test_kernel(PairArgs a) {
  const int nbk = a.nbx * a.nby;
  for (int bk = blockIdx.x; bk < nbk; bk += gridDim.x) {
    const int s = a.start[bk], e = a.start[bk + 1], m = e - s;
    const long long np = (long long)m * (m - 1) / 2;
    const int bi = bk / a.nby, bj = bk % a.nby;
    for (long long t = threadIdx.x; t < np; t += blockDim.x) {
      // t -> (u, v), u < v
      int u = (int)((sqrt(8.0 * (double)t + 1.0) - 1.0) / 2.0) + 1;
      while ((long long)u * (u - 1) / 2 > t) --u;
      while ((long long)(u + 1) * u / 2 <= t) ++u;
      const int v = (int)(t - (long long)u * (u - 1) / 2);
      int p = a.list[s + u], q = a.list[s + v];
      if (p > q) { const int w = p; p = q; q = w; }
      const double* b1 = a.box + 4 * (long long)p;
      const double* b2 = a.box + 4 * (long long)q;
      bool hit;
      if (a.mode == 0) {  // overlap with eps (check.py:64-66)
        const double eps = 1e-9;
        hit = b1[0] < b2[1] - eps && b2[0] < b1[1] - eps && b1[2] < b2[3] - eps &&
              b2[2] < b1[3] - eps;
      } else {  // terminal spacing: boxes overlap and max(dx, dy) < min_cc - tol (check.py:130-139)
        const double eps = 1e-9;
        const bool ov = b1[0] < b2[1] - eps && b2[0] < b1[1] - eps && b1[2] < b2[3] - eps &&
                        b2[2] < b1[3] - eps;
        const double dx = fabs(b1[0] - b2[0]), dy = fabs(b1[2] - b2[2]);
        hit = ov && fmax(dx, dy) < a.min_cc - a.tol;
      }
      if (!hit) continue;
      // report from the bucket of the intersection's lower-left corner only
      const int ci = bucket_of(fmax(b1[0], b2[0]), a.bucket, a.nbx);
      const int cj = bucket_of(fmax(b1[2], b2[2]), a.bucket, a.nby);
      if (ci != bi || cj != bj) continue;
      const int slot = atomicAdd(a.n_out, 1);
      if (slot < a.cap_out) {
        a.out[2 * slot] = p;
        a.out[2 * slot + 1] = q;
      }
    }
  }
}

}  // namespace

void launch_rebalance(const RebalanceArgs& a, cudaStream_t s) {
  rebalance_kernel<<<1, kRbThreads, 0, s>>>(a);
}

void launch_check(const CheckArgs& a, cudaStream_t s) {
  check_inst_kernel<<<grid_blocks(a.n_inst, 256, kMaxBlocks), 256, 0, s>>>(a);
  if (a.n_net > 0) check_net_kernel<<<grid_blocks(a.n_net, 256, kMaxBlocks), 256, 0, s>>>(a);
}

void launch_pair_count(const PairArgs& a, cudaStream_t s) {
  pair_count_kernel<<<grid_blocks(a.n, 256, kMaxBlocks), 256, 0, s>>>(a);
}
void launch_pair_fill(const PairArgs& a, cudaStream_t s) {
  pair_fill_kernel<<<grid_blocks(a.n, 256, kMaxBlocks), 256, 0, s>>>(a);
}
void launch_pair_test(const PairArgs& a, cudaStream_t s) {
  const int nbk = a.nbx * a.nby;
  pair_test_kernel<<<nbk < 4096 ? nbk : 4096, 256, 0, s>>>(a);
}

}  // namespace p3d
