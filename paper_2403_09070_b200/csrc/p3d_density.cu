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
#include <limits.h>

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

// ---------------------------------------------------------------------------
// Spatially ordered, shared-memory-privatised scatter (the fused loop's K2).
// Every P3D_RESORT_EVERY-th iteration the non-macro objects are counting-sorted
// by the planar tile (kTile x kTile bins) of their current centre (in between,
// the last sort's order is reused); a CTA then takes 1024
// consecutive objects of that order, whose footprints cover a small bounding
// box of bins: it accumulates their int64 terms in shared memory (contention
// moves from L2 atomics to shared-memory atomics) and flushes the box once.
// Boxes that do not fit fall back to global atomics.  Integer sums make the
// map independent of the (atomic, unstable) order within a tile.
// ---------------------------------------------------------------------------
constexpr int kTile = 16;
#ifndef P3D_CHUNK
#define P3D_CHUNK 1024
#endif
constexpr int kChunk = P3D_CHUNK;  // records per scatter CTA
#ifndef P3D_MACRO_SPLIT
#define P3D_MACRO_SPLIT 1
#endif
constexpr int kMacroSplit = P3D_MACRO_SPLIT;  // CTAs per macro footprint in the scatter
constexpr int kBoxBins = 6144;  // 48 KB of int64 bins per CTA

// exclusive scan of the tile histogram by one block; re-zeroes the histogram
__device__ __forceinline__ void scan_tiles(const TileSort& ts) {
  __shared__ int carry;
  __shared__ int wsum[32];
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  const int nw = blockDim.x >> 5;
  for (int base = 0; base < ts.n_tiles; base += blockDim.x) {
    const int t = base + threadIdx.x;
    const int v = t < ts.n_tiles ? ((volatile int*)ts.hist)[t] : 0;
    int x = v;  // inclusive warp scan
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) wsum[wid] = x;
    __syncthreads();
    if (wid == 0) {
      int w = lane < nw ? wsum[lane] : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, w, o);
        if (lane >= o) w += y;
      }
      wsum[lane] = w;
    }
    __syncthreads();
    const int excl = carry + (wid ? wsum[wid - 1] : 0) + x - v;
    if (t < ts.n_tiles) {
      ts.start[t] = excl;
      ts.cursor[t] = excl;
      ts.hist[t] = 0;
    }
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) carry = excl + v;
    __syncthreads();
  }
  if (threadIdx.x == 0) ts.start[ts.n_tiles] = carry;
}

#ifndef P3D_RESORT_EVERY
#define P3D_RESORT_EVERY 8
#endif
#ifndef P3D_SCATTER_DIRECT
#define P3D_SCATTER_DIRECT 1
#endif
#ifndef P3D_SCATTER_SZREC
#define P3D_SCATTER_SZREC 1  // sort records hold both dies' sizes (see chunk_charge)
#endif
#ifndef P3D_SCATTER_CELL
#define P3D_SCATTER_CELL 1
#endif
__device__ __forceinline__ bool resort_now(const TileSort& ts) {
  if (!ts.perm || !ts.it || ts.every <= 1) return true;
  return !*(volatile const int32_t*)ts.valid || (*ts.it % ts.every) == 0;
}
// the decision as the histogram pass took it (place / scatter: valid may have
// been set by then, so they must not re-evaluate resort_now)
__device__ __forceinline__ bool resort_decided(const TileSort& ts) {
  return ts.decision ? *(volatile const int32_t*)ts.decision != 0 : resort_now(ts);
}

// K2 step 1: per-object tile of the centre + tile histogram; the last block
// scans the histogram.  The first n_macro * kMacroSplit blocks scatter the macros
// (per-macro footprint tile, int64 global atomics), independent of the sort.
template <class Cloud>
__global__ void __launch_bounds__(256) tile_hist_kernel(Cloud cl, int n, p3d_grid g, TileSort ts,
                                                       const int32_t* macro_ids, int n_macro,
                                                       unsigned long long* rho, const int* halt) {
  pdl_wait();
  if (halt && *halt) return;
  extern __shared__ int sh_hist[];
  // the same value in every CTA: valid and it change only in later kernels
  const bool sort = resort_now(ts);
  if ((int)blockIdx.x < n_macro * kMacroSplit) {  // kMacroSplit CTAs per macro footprint
    scatter_object_block(cl.get(macro_ids[blockIdx.x / kMacroSplit]), g, rho,
                         blockIdx.x % kMacroSplit, kMacroSplit);
  } else if (sort) {
    for (int t = threadIdx.x; t < ts.n_tiles; t += blockDim.x) sh_hist[t] = 0;
    __syncthreads();
    // the tile of an object's centre only groups the records (any assignment
    // is exact: a footprint outside its CTA's window goes to global atomics),
    // so the centre is scaled by reciprocals, and only x, y and the macro
    // flag are read
    const double rtw = 1.0 / (g.wb * kTile), rth = 1.0 / (g.hb * kTile);
    const int b = blockIdx.x - n_macro * kMacroSplit, nb = gridDim.x - n_macro * kMacroSplit;
    for (int k = b * blockDim.x + threadIdx.x; k < n; k += nb * blockDim.x) {
      const int i = k < ts.ni ? ts.i0 + k : ts.f0 + (k - ts.ni);  // this rank's objects
      const double cx = cl.cx(i), cy = cl.cy(i);
      if (cl.is_macro(i)) {
        ts.tile_of[k] = -1;
        continue;
      }
      int tx = (int)floor(cx * rtw), ty = (int)floor(cy * rth);
      tx = tx < 0 ? 0 : (tx >= ts.tiles_x ? ts.tiles_x - 1 : tx);
      ty = ty < 0 ? 0 : (ty >= ts.tiles_y ? ts.tiles_y - 1 : ty);
      const int t = tx * ts.tiles_y + ty;
      ts.tile_of[k] = t;
      atomicAdd(&sh_hist[t], 1);
    }
    __syncthreads();
    for (int t = threadIdx.x; t < ts.n_tiles; t += blockDim.x)
      if (sh_hist[t]) atomicAdd(&ts.hist[t], sh_hist[t]);
  }
  if (!sort) {  // nothing to scan: no ticket (most CTAs exit at once); CTA 0 records it
    if (blockIdx.x == 0 && threadIdx.x == 0 && ts.decision) *ts.decision = 0;
    return;
  }
  if (last_block_all(ts.counter)) {
    if (ts.decision && threadIdx.x == 0) *ts.decision = 1;
    scan_tiles(ts);
  }
}

// Stable-per-block placement: each CTA ranks its objects per tile in shared
// memory, reserves one range per (CTA, tile) with a single global atomic, and
// writes each object's charge record (x, y, z, w, h, weight) at its slot, so
// the scatter reads its chunk contiguously.
constexpr int kPlacePerThread = 8;

template <class Cloud>
__global__ void __launch_bounds__(256) tile_place_kernel(Cloud cl, int n, TileSort ts,
                                                        const int* halt) {
  pdl_wait();
  if (halt && *halt) return;
  const bool sorting = resort_decided(ts);
#if P3D_SCATTER_DIRECT
  if (!sorting) return;  // the scatter reads the objects through perm itself
#endif
  if (!sorting) {
    // refresh the records in the last sort's order (coalesced record writes)
    const int total = ts.start[ts.n_tiles];
    for (int pos = blockIdx.x * blockDim.x + threadIdx.x; pos < total;
         pos += gridDim.x * blockDim.x) {
      const int kl = ts.perm[pos];
      const int i = kl < ts.ni ? ts.i0 + kl : ts.f0 + (kl - ts.ni);
      const Charge q = cl.get(i);
      double2* r = reinterpret_cast<double2*>(ts.rec) + 3 * (long long)pos;
      r[0] = make_double2(q.x, q.y);
      r[1] = make_double2(q.z, q.w);
      r[2] = make_double2(q.h, q.weight);
    }
    return;
  }
  extern __shared__ int sh[];
  int* cnt = sh;                  // [n_tiles]
  int* base = sh + ts.n_tiles;    // [n_tiles]
  for (int t = threadIdx.x; t < ts.n_tiles; t += blockDim.x) cnt[t] = 0;
  __syncthreads();
  const int i0 = blockIdx.x * blockDim.x * kPlacePerThread + threadIdx.x;
  int tile[kPlacePerThread], rank[kPlacePerThread];
#pragma unroll
  for (int k = 0; k < kPlacePerThread; ++k) {
    const int i = i0 + k * blockDim.x;
    tile[k] = i < n ? ts.tile_of[i] : -1;
    rank[k] = tile[k] >= 0 ? atomicAdd(&cnt[tile[k]], 1) : 0;
  }
  __syncthreads();
  for (int t = threadIdx.x; t < ts.n_tiles; t += blockDim.x)
    base[t] = cnt[t] ? atomicAdd(&ts.cursor[t], cnt[t]) : 0;
  __syncthreads();
#pragma unroll
  for (int k = 0; k < kPlacePerThread; ++k) {
    if (tile[k] < 0) continue;
    const int kl = i0 + k * blockDim.x;
    const int i = kl < ts.ni ? ts.i0 + kl : ts.f0 + (kl - ts.ni);  // this rank's objects
    const int pos = base[tile[k]] + rank[k];
#if P3D_SCATTER_CELL
    const Charge q = cl.get_nonmacro(i);  // tile >= 0: not a macro
#else
    const Charge q = cl.get(i);
#endif
    ts.order[pos] = tile[k];
    if (ts.perm) ts.perm[pos] = kl;
    double2* r = reinterpret_cast<double2*>(ts.rec) + 3 * (long long)pos;
#if P3D_SCATTER_SZREC
    if (ts.perm) {  // the record holds the sizes of both dies: the scatter reads the
      (void)q;      // centre through perm and picks the die's pair itself
      if (i < cl.n_inst) {
        r[0] = make_double2(cl.wt[i], cl.ht[i]);
        r[1] = make_double2(cl.wb[i], cl.hb[i]);
      } else {
        const int f = i - cl.n_inst;
        r[0] = r[1] = make_double2(cl.fw[f], cl.fh[f]);
      }
      continue;
    }
#endif
    r[0] = make_double2(q.x, q.y);
    r[1] = make_double2(q.z, q.w);
    r[2] = make_double2(q.h, q.weight);
  }
  if (ts.valid && blockIdx.x == 0 && threadIdx.x == 0) *ts.valid = 1;
}

__device__ __forceinline__ Charge rec_charge(const TileSort& ts, int pos, double dep) {
  const double2* r = reinterpret_cast<const double2*>(ts.rec) + 3 * (long long)pos;
  const double2 a = r[0], b = r[1], c = r[2];
  Charge q;
  q.x = a.x; q.y = a.y; q.z = b.x; q.w = b.y; q.h = c.x; q.weight = c.y; q.dep = dep;
  return q;
}

// One fixed-point term into the CTA's shared-memory window (int64 bins as
// two u32 halves: 32-bit shared atomics, native ATOMS.ADD, with the carry
// propagated by the thread that produced it — exact), or straight to the
// global map when it falls outside the window.
#ifndef P3D_PUT_NOBRANCH
#define P3D_PUT_NOBRANCH 1
#endif
struct SmemWindow {
  unsigned int *lo32, *hi32;
  int X0, Y0, W, H, nz;
  bool local;
};

__device__ __forceinline__ void put_term(const SmemWindow& w, const p3d_grid& g,
                                         unsigned long long* rho, long long t, int ix, int iy,
                                         int iz) {
#if !P3D_PUT_NOBRANCH
  if (!t) return;
#endif
  const int lx = ix - w.X0, ly = iy - w.Y0;
  if (w.local && (unsigned)lx < (unsigned)w.W && (unsigned)ly < (unsigned)w.H) {
    const int b = (lx * w.H + ly) * w.nz + iz;
    const unsigned int tl = (unsigned int)t, th = (unsigned int)((unsigned long long)t >> 32);
    const unsigned int old = atomicAdd(&w.lo32[b], tl);
    const unsigned int hadd = th + (old + tl < old ? 1u : 0u);
#if P3D_PUT_NOBRANCH  // the high half is almost never 0: no branch (adding 0 is exact)
    atomicAdd(&w.hi32[b], hadd);
#else
    if (hadd) atomicAdd(&w.hi32[b], hadd);
#endif
  } else {
    atomicAdd(rho + ((long long)(ix * g.ny + iy) * g.nz + iz), (unsigned long long)t);
  }
}

// all terms of one object: per-axis overlap lengths computed once; footprints
// of at most 3 x 3 x 2 bins fully unrolled (same terms as scatter_object)
template <int MX, int MY, int MZ>
__device__ __forceinline__ void scatter_small(const Charge& q, const p3d_grid& g,
                                              const SmemWindow& w, unsigned long long* rho,
                                              const Footprint& f, int nxr, int nyr, int nzr) {
  double wx[MX], wy[MY], wz[MZ];
  axis_weights<MX>(f.ax, g.wb, wx);
  axis_weights<MY>(f.ay, g.hb, wy);
  axis_weights<MZ>(f.az, g.db, wz);
#pragma unroll
  for (int x = 0; x < MX; ++x)
#pragma unroll
    for (int y = 0; y < MY; ++y) {
      const double wxy = wx[x] * wy[y];
#pragma unroll
      for (int z = 0; z < MZ; ++z)
        if (x < nxr && y < nyr && z < nzr) {
          const double vol = wxy * wz[z];
          put_term(w, g, rho, __double2ll_rn((q.weight * vol) * g.fx_scale), f.ax.i0 + x,
                   f.ay.i0 + y, f.az.i0 + z);
        }
    }
}

#ifndef P3D_SCATTER_SMALL2
#define P3D_SCATTER_SMALL2 0  // measured: K2 +1.3 us with it (K4 -4 us with its own)
#endif
__device__ __forceinline__ void scatter_terms(const Charge& q, const p3d_grid& g,
                                              const SmemWindow& w, unsigned long long* rho) {
  const Footprint f = footprint(q, g);
  const int nxr = f.ax.i1 - f.ax.i0 + 1, nyr = f.ay.i1 - f.ay.i0 + 1, nzr = f.az.i1 - f.az.i0 + 1;
  // optional 2 x 2 x 2 path (every cell and filler of the BASELINE configs)
#if P3D_SCATTER_SMALL2
  if (nxr <= 2 && nyr <= 2 && nzr <= 2) {
    scatter_small<2, 2, 2>(q, g, w, rho, f, nxr, nyr, nzr);
    return;
  }
#endif
  if (nxr <= 3 && nyr <= 3 && nzr <= 2) {
    scatter_small<3, 3, 2>(q, g, w, rho, f, nxr, nyr, nzr);
    return;
  }
  for (int ix = f.ax.i0; ix <= f.ax.i1; ++ix) {
    const double wx = overlap_len(f.ax, ix, g.wb);
    for (int iy = f.ay.i0; iy <= f.ay.i1; ++iy) {
      const double wxy = wx * overlap_len(f.ay, iy, g.hb);
      for (int iz = f.az.i0; iz <= f.az.i1; ++iz) {
        const double vol = wxy * overlap_len(f.az, iz, g.db);
        put_term(w, g, rho, __double2ll_rn((q.weight * vol) * g.fx_scale), ix, iy, iz);
      }
    }
  }
}

// the k-th charge of the sorted order: its record, or (between re-sorts, with
// P3D_SCATTER_DIRECT) the object itself through the last sort's permutation
__device__ __forceinline__ Charge chunk_charge(const TileSort& ts, const CloudGP& cl, bool direct,
                                               int k, double dep) {
#if P3D_SCATTER_SZREC
  if (ts.perm) {  // every iteration: perm + the sorted sizes, then the centre
    const int kl = ts.perm[k];
    const double2* r = reinterpret_cast<const double2*>(ts.rec) + 3 * (long long)k;
    const double2 s0 = r[0], s1 = r[1];
    const int i = kl < ts.ni ? ts.i0 + kl : ts.f0 + (kl - ts.ni);
    return cl.get_sized(i, s0, s1);
  }
#endif
#if P3D_SCATTER_DIRECT
  if (direct) {
    const int kl = ts.perm[k];
    const int i = kl < ts.ni ? ts.i0 + kl : ts.f0 + (kl - ts.ni);
#if P3D_SCATTER_CELL
    return cl.get_nonmacro(i);  // perm holds no macro (their tile is -1)
#else
    return cl.get(i);
#endif
  }
#endif
  return rec_charge(ts, k, dep);
}

__global__ void __launch_bounds__(256) scatter_tiled_kernel(p3d_grid g, TileSort ts, CloudGP cl,
                                                           unsigned long long* rho,
                                                           const int* halt) {
  pdl_wait();
  if (halt && *halt) return;
  const bool direct = !resort_decided(ts);
  extern __shared__ unsigned int sbin32[];
  __shared__ int box[4];
  const int total = ts.start[ts.n_tiles];
  const int c0 = blockIdx.x * kChunk;
  if (c0 >= total) return;
  const int c1 = min(total, c0 + kChunk);
  const double dep = g.dz / 2;
  // window: the chunk's tiles (when they share one tile column) widened by the
  // footprint margin; otherwise the bounding box of the chunk's footprints
  const int tf = ts.order[c0], tl = ts.order[c1 - 1];
  SmemWindow w;
  w.nz = g.nz;
  if (tf / ts.tiles_y == tl / ts.tiles_y) {
    const int tx = tf / ts.tiles_y;
    w.X0 = max(0, tx * kTile - ts.margin);
    const int X1 = min(g.nx - 1, tx * kTile + kTile - 1 + ts.margin);
    w.Y0 = max(0, (tf % ts.tiles_y) * kTile - ts.margin);
    const int Y1 = min(g.ny - 1, (tl % ts.tiles_y) * kTile + kTile - 1 + ts.margin);
    w.W = X1 - w.X0 + 1;
    w.H = Y1 - w.Y0 + 1;
  } else {
    int bx0 = INT_MAX, bx1 = -1, by0 = INT_MAX, by1 = -1;
    for (int k = c0 + threadIdx.x; k < c1; k += blockDim.x) {
      const Footprint f = footprint(chunk_charge(ts, cl, direct, k, dep), g);
      bx0 = min(bx0, f.ax.i0); bx1 = max(bx1, f.ax.i1);
      by0 = min(by0, f.ay.i0); by1 = max(by1, f.ay.i1);
    }
    if (threadIdx.x == 0) { box[0] = INT_MAX; box[1] = -1; box[2] = INT_MAX; box[3] = -1; }
    __syncthreads();
    atomicMin(&box[0], bx0); atomicMax(&box[1], bx1);
    atomicMin(&box[2], by0); atomicMax(&box[3], by1);
    __syncthreads();
    w.X0 = box[0];
    w.Y0 = box[2];
    w.W = box[1] - box[0] + 1;
    w.H = box[3] - box[2] + 1;
  }
  const int nbins = w.W * w.H * w.nz;
  w.local = (long long)w.W * w.H * w.nz <= kBoxBins;
  w.lo32 = sbin32;
  w.hi32 = sbin32 + kBoxBins;
  if (w.local) {
    for (int b = threadIdx.x; b < nbins; b += blockDim.x) w.lo32[b] = w.hi32[b] = 0u;
    __syncthreads();
  }
  for (int k = c0 + threadIdx.x; k < c1; k += blockDim.x)
    scatter_terms(chunk_charge(ts, cl, direct, k, dep), g, w, rho);
  if (!w.local) return;
  __syncthreads();
#if P3D_PUT_NOBRANCH
  // one (x, y) column of nz bins per thread and step: one division per column
  for (int r = threadIdx.x; r < w.W * w.H; r += blockDim.x) {
    const int ix = r / w.H, iy = r - ix * w.H;
    unsigned long long* dst = rho + ((long long)((ix + w.X0) * g.ny + (iy + w.Y0)) * g.nz);
    for (int iz = 0; iz < w.nz; ++iz) {
      const int b = r * w.nz + iz;
      const unsigned long long v = ((unsigned long long)w.hi32[b] << 32) | w.lo32[b];
      if (v) atomicAdd(dst + iz, v);
    }
  }
#else
  for (int b = threadIdx.x; b < nbins; b += blockDim.x) {
    const unsigned long long v = ((unsigned long long)w.hi32[b] << 32) | w.lo32[b];
    if (!v) continue;
    const int iz = b % w.nz, r = b / w.nz, iy = r % w.H, ix = r / w.H;
    atomicAdd(rho + ((long long)((ix + w.X0) * g.ny + (iy + w.Y0)) * g.nz + iz), v);
  }
#endif
}

void tiled_scatter_setup() {
  static bool done_dev[kMaxDevices] = {};  // function attributes are per device
  bool& done = done_dev[current_device()];
  if (done) return;
  cudaFuncSetAttribute(scatter_tiled_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       kBoxBins * 8);
  cudaFuncSetAttribute(tile_place_kernel<CloudGP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       200 * 1024);
  cudaFuncSetAttribute(tile_hist_kernel<CloudGP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       200 * 1024);
  done = true;
}

int tiled_scatter_tiles(const p3d_grid& g, int* tx, int* ty) {
  *tx = (g.nx + kTile - 1) / kTile;
  *ty = (g.ny + kTile - 1) / kTile;
  return *tx * *ty;
}

void launch_scatter_tiled(const CloudGP& cl, int n, int n_macro, const int32_t* macro_ids,
                          const p3d_grid& g, const TileSort& ts, int64_t* rho, const int* halt,
                          cudaStream_t s) {
  unsigned long long* r = reinterpret_cast<unsigned long long*>(rho);
  const int nb = grid_blocks(n, 256, 148 * 8);
  pdl_launch_tag(4, tile_hist_kernel<CloudGP>, n_macro * kMacroSplit + nb, 256, ts.n_tiles * sizeof(int), s, cl, n, g,
             ts, macro_ids, n_macro, r, halt);
  const int np = (n + 256 * kPlacePerThread - 1) / (256 * kPlacePerThread);
  pdl_launch_tag(4, tile_place_kernel<CloudGP>, np, 256, 2 * ts.n_tiles * sizeof(int), s, cl, n, ts, halt);
  const int chunks = (n + kChunk - 1) / kChunk;
  pdl_launch_tag(4, scatter_tiled_kernel, chunks, 256, kBoxBins * 8, s, g, ts, cl, r, halt);
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
// exact energy gradient (density_energy_and_gradient, density.py:389-565):
// cells differentiate the overlap volume through the two face columns of each
// axis, macros differentiate their corner stamps against the suffix-summed
// potential.  Same terms, same order as the reference (compiled -fmad=false).
// ---------------------------------------------------------------------------
// inclusive sums toward smaller indices along one axis (density.py:212-217)
__global__ void suffix_axis_kernel(const double* in, double* out, int nx, int ny, int nz,
                                   int axis) {
  const int len = axis == 0 ? nx : (axis == 1 ? ny : nz);
  const long long stride = axis == 0 ? (long long)ny * nz : (axis == 1 ? nz : 1);
  const long long n_lines = (long long)nx * ny * nz / len;
  for (long long l = blockIdx.x * (long long)blockDim.x + threadIdx.x; l < n_lines;
       l += (long long)gridDim.x * blockDim.x) {
    long long base;
    if (axis == 0) base = l;
    else if (axis == 1) base = (l / nz) * (long long)ny * nz + (l % nz);
    else base = l * nz;
    double s = 0.0;
    for (int i = len - 1; i >= 0; --i) {
      s += in[base + i * stride];
      out[base + i * stride] = s;
    }
  }
}

// density.py:389-441, one cell: d/d(center) of sum_b phi_b vol(D cap b)
__device__ __forceinline__ void cell_face_grad(const Footprint& f, const p3d_grid& g,
                                               const double* phi, double (&out)[3]) {
  const AxisSpan ax[3] = {f.ax, f.ay, f.az};
  const double steps[3] = {g.wb, g.hb, g.db};
  const int nb[3] = {g.nx, g.ny, g.nz};
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    long long fh = (long long)floor(ax[a].hi / steps[a]), fl = (long long)floor(ax[a].lo / steps[a]);
    fh = fh < 0 ? 0 : (fh > nb[a] - 1 ? nb[a] - 1 : fh);
    fl = fl < 0 ? 0 : (fl > nb[a] - 1 ? nb[a] - 1 : fl);
    const int o1 = a == 0 ? 1 : 0, o2 = a == 2 ? 1 : 2;
    double acc = 0.0;
    for (int b1 = ax[o1].i0; b1 <= ax[o1].i1; ++b1) {
      const double w1 = overlap_len(ax[o1], b1, steps[o1]);
      for (int b2 = ax[o2].i0; b2 <= ax[o2].i1; ++b2) {
        const double w12 = w1 * overlap_len(ax[o2], b2, steps[o2]);
        int ih[3], il[3];
        ih[o1] = il[o1] = b1;
        ih[o2] = il[o2] = b2;
        ih[a] = (int)fh;
        il[a] = (int)fl;
        const double ph = phi[((long long)ih[0] * g.ny + ih[1]) * g.nz + ih[2]];
        const double pl = phi[((long long)il[0] * g.ny + il[1]) * g.nz + il[2]];
        acc += (ph - pl) * w12;
      }
    }
    out[a] = acc;
  }
}

// one corner's trilinear stamp dotted with the suffix map (density.py:505-530);
// axis >= 0 differentiates the stamp along that axis (density.py:466-476)
__device__ __forceinline__ double corner_stamp(const p3d_grid& g, const double* sphi,
                                               const double (&c)[3], int axis) {
  const double steps[3] = {g.wb, g.hb, g.db};
  const int nb[3] = {g.nx, g.ny, g.nz};
  long long i0[3];
  double v[3][2];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const double base = c[a] / steps[a];
    i0[a] = (long long)floor(base);
    const double frac = base - (double)i0[a];
    if (a == axis) {
      v[a][0] = -1.0 / steps[a];
      v[a][1] = 1.0 / steps[a];
    } else {
      v[a][0] = 1.0 - frac;
      v[a][1] = frac;
    }
  }
  double acc = 0.0;
  for (int b0 = 0; b0 < 2; ++b0) {
    const long long g0 = i0[0] + b0;
    if (g0 < 0 || g0 >= nb[0]) continue;
    for (int b1 = 0; b1 < 2; ++b1) {
      const long long g1 = i0[1] + b1;
      if (g1 < 0 || g1 >= nb[1]) continue;
      for (int b2 = 0; b2 < 2; ++b2) {
        const long long g2 = i0[2] + b2;
        if (g2 < 0 || g2 >= nb[2]) continue;
        const double val = sphi[(g0 * g.ny + g1) * g.nz + g2];
        acc += val * ((v[0][b0] * v[1][b1]) * v[2][b2]);  // density.py:527-528
      }
    }
  }
  return acc;
}

// density.py:444-486 (gradient) and 489-502 (phibar) of one macro
__device__ __forceinline__ void macro_face_grad(const Charge& q, const p3d_grid& g,
                                                const double* sphi, double (&grad)[3],
                                                double& phibar) {
  const double ext[3] = {g.dx, g.dy, g.dz};
  const double half[3] = {q.w / 2, q.h / 2, q.dep / 2};
  const double cen[3] = {q.x, q.y, q.z};
  double pacc = 0.0;
  double gacc[3] = {0.0, 0.0, 0.0};
  for (int s = 0; s < 8; ++s) {
    const double sg[3] = {(s & 4) ? 1.0 : -1.0, (s & 2) ? 1.0 : -1.0, (s & 1) ? 1.0 : -1.0};
    const double sign = -sg[0] * sg[1] * sg[2];
    double c[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) c[a] = clipd(cen[a] + sg[a] * half[a], 0.0, ext[a]);
    pacc += sign * corner_stamp(g, sphi, c, -1);
  }
  // the reference accumulates per axis over the 8 corners and every stamp point
  for (int axis = 0; axis < 3; ++axis) {
    double acc = 0.0;
    for (int s = 0; s < 8; ++s) {
      const double sg[3] = {(s & 4) ? 1.0 : -1.0, (s & 2) ? 1.0 : -1.0, (s & 1) ? 1.0 : -1.0};
      const double sign = -sg[0] * sg[1] * sg[2];
      double c[3];
#pragma unroll
      for (int a = 0; a < 3; ++a) c[a] = clipd(cen[a] + sg[a] * half[a], 0.0, ext[a]);
      const double steps[3] = {g.wb, g.hb, g.db};
      const int nb[3] = {g.nx, g.ny, g.nz};
      long long i0[3];
      double v[3][2];
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        const double base = c[a] / steps[a];
        i0[a] = (long long)floor(base);
        const double frac = base - (double)i0[a];
        if (a == axis) { v[a][0] = -1.0 / steps[a]; v[a][1] = 1.0 / steps[a]; }
        else { v[a][0] = 1.0 - frac; v[a][1] = frac; }
      }
      for (int b0 = 0; b0 < 2; ++b0) {
        const long long g0 = i0[0] + b0;
        if (g0 < 0 || g0 >= nb[0]) continue;
        for (int b1 = 0; b1 < 2; ++b1) {
          const long long g1 = i0[1] + b1;
          if (g1 < 0 || g1 >= nb[1]) continue;
          for (int b2 = 0; b2 < 2; ++b2) {
            const long long g2 = i0[2] + b2;
            if (g2 < 0 || g2 >= nb[2]) continue;
            const double val = sphi[(g0 * g.ny + g1) * g.nz + g2];
            acc += sign * val * ((v[0][b0] * v[1][b1]) * v[2][b2]);  // density.py:484
          }
        }
      }
    }
    gacc[axis] = acc * g.bin_vol;
  }
  for (int a = 0; a < 3; ++a) grad[a] = gacc[a];
  phibar = pacc * g.bin_vol / fmax(q.w * q.h * q.dep, 1e-300);
}

__global__ void __launch_bounds__(256) energy_grad_kernel(CloudArrays cl, p3d_grid g,
                                                         const double* phi, const double* sphi,
                                                         const uint8_t* freeze, double* grad,
                                                         double* partials, unsigned int* counter,
                                                         double* energy) {
  __shared__ double red[32];
  double e[1] = {0.0};
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < cl.c.n; i += gridDim.x * blockDim.x) {
    const Charge q = cl.get(i);
    double gr[3], pb;
    if (cl.is_macro(i)) {
      macro_face_grad(q, g, sphi, gr, pb);
    } else {
      const Footprint f = footprint(q, g);
      double tot = 0.0, a = 0.0;
      for (int ix = f.ax.i0; ix <= f.ax.i1; ++ix) {  // density.py:376-386 on phi alone
        const double wx = overlap_len(f.ax, ix, g.wb);
        for (int iy = f.ay.i0; iy <= f.ay.i1; ++iy) {
          const double wxy = wx * overlap_len(f.ay, iy, g.hb);
          for (int iz = f.az.i0; iz <= f.az.i1; ++iz) {
            const double vol = wxy * overlap_len(f.az, iz, g.db);
            tot += vol;
            a += phi[((long long)ix * g.ny + iy) * g.nz + iz] * vol;
          }
        }
      }
      pb = a / fmax(tot, 1e-300);
      cell_face_grad(f, g, phi, gr);
    }
    const double w2 = 2.0 * q.weight;
    grad[3 * i + 0] = gr[0] * w2;
    grad[3 * i + 1] = gr[1] * w2;
    grad[3 * i + 2] = (freeze && freeze[i]) ? 0.0 : gr[2] * w2;
    e[0] += charge_of(q) * pb;
  }
  block_sum<1>(e, red);
  if (threadIdx.x == 0) partials[blockIdx.x] = e[0];
  if (last_block(counter)) {
    const double s = ordered_sum(partials, gridDim.x, red);
    if (threadIdx.x == 0) *energy = s;
  }
}

void launch_energy_grad(const p3d_cloud& c, const p3d_grid& g, const double* phi,
                        const uint8_t* freeze, double* energy, double* grad, double* scratch,
                        cudaStream_t s) {
  CloudArrays cl;
  cl.c = c;
  const long long B = (long long)g.nx * g.ny * g.nz;
  double* sphi = scratch;  // [B]
  unsigned int* counter = reinterpret_cast<unsigned int*>(scratch + B);
  double* partials = scratch + B + 8;
  const int lb = (int)((B + 255) / 256 > 1024 ? 1024 : (B + 255) / 256);
  if (c.n_macro > 0) {
    suffix_axis_kernel<<<lb, 256, 0, s>>>(phi, sphi, g.nx, g.ny, g.nz, 0);
    suffix_axis_kernel<<<lb, 256, 0, s>>>(sphi, sphi, g.nx, g.ny, g.nz, 1);
    suffix_axis_kernel<<<lb, 256, 0, s>>>(sphi, sphi, g.nx, g.ny, g.nz, 2);
  }
  const int nb = grid_blocks(c.n, 256, 1024);
  energy_grad_kernel<<<nb, 256, 0, s>>>(cl, g, phi, sphi, freeze, grad, partials, counter, energy);
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
    const long long s = block_sum_ll_partials((volatile long long*)partials, gridDim.x);
    if (threadIdx.x == 0) *out = (double)s * scale;
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
