// Internal launch-argument blocks and launcher declarations shared by the
// translation units of libp3d.so.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/p3d.h"

namespace p3d {

constexpr int kMaxBlocks = 2048;      // cap on grid-stride grids (partials sizing)
constexpr int kPartialStride = 8 * kMaxBlocks;

// partials layout inside p3d_gp::partials ([16][kPartialStride] doubles)
enum PartialSlot {
  kSlotNet = 0,      // net kernel: 6 x blocks
  kSlotGather = 1,   // owner gather: 3 x blocks
  kSlotOvfl = 2,     // overflow
  kSlotDens = 3,     // density gather (energy, |dens|, |wl|)
  kSlotStep = 4,     // preconditioner / BB norms
  kSlotGeneric = 5,  // generic (high-degree) nets
  kSlotAdv = 6,      // advance: |v_new - v|^2
  kSlotFinal = 15,   // finalised scalars of the sub-kernels
};
// offsets inside the final slot
enum FinalIdx {
  kFinNet = 0,      // 6 values: planar x, planar y, cut, exact x, exact y, crossings
  kFinNorm = 8,     // 4 values: |gx|, |gy|, |gzb|, Eq. 17 scale
  kFinOvfl = 16,    // 1 value: overflow excess (already / movable volume)
  kFinGeneric = 24, // 6 values: generic-net totals
};
// counters inside p3d_loop_state::counters
enum CounterIdx { kCntNet = 0, kCntGather, kCntOvfl, kCntDens, kCntStep, kCntAdvance, kCntOp, kCntGeneric, kCntTile };

struct NetArgs {
  int n_net, blocks;
  const int32_t* net_ptr;
  const int32_t* pin_inst;
  const int32_t* net_order;
  const uint8_t* net_dup;
  const int32_t* pin_slot;
  double gamma, scale4;
  const double* gamma_ptr;    // nullable: device gamma overrides `gamma`
  int want_pins, value_mode;
  double* out4;  // [n_pin][4] by slot (fused) or nullptr
  double *gx, *gy, *gc, *gb;  // separate per-pin outputs (per-op)
  double* partials;           // [6][blocks]
  unsigned int* counter;
  double* final6;             // nullable: skip reduction
  double* value_out;          // nullable
  const int* halt;            // nullable: skip when *halt != 0
};

struct GatherArgs {
  int n_obj, blocks;
  const int32_t* obj_slot_ptr;
  const double* pin4;
  double* out;           // [4][n_obj]
  double* partials;      // [3][blocks]
  unsigned int* counter;
  double* final_norms;   // nullable: 4 values
  const int* halt;
};

// K1 fused-loop variant (p3d_wl_fused.cu): degree-bucketed transposed pins
struct FusedNetArgs {
  int n_net, blocks;
  int n_tasks;                // warp tasks
  int task_rank, task_size;   // this rank takes tasks w % task_size == task_rank (sharded)
  const int4* tasks;          // (pin base, bucket size, first net in bucket, degree | 0 = generic)
  const int32_t* task_t0;     // permuted index of the bucket's first net
  int n_generic;              // nets of degree outside [2, 6]
  const int32_t* generic_nets;  // their permuted indices
  double* gpartials;
  unsigned int* gcounter;
  double* generic6;           // their 6 totals (read by the staged kernel's epilogue)
  const int32_t* net_base;    // [n_net] first pin index of the net (permuted order)
  const int32_t* net_deg;     // [n_net]
  const int32_t* net_stride;  // [n_net] distance between consecutive pins of a net
  const uint8_t* net_dup;     // [n_net] permuted: bit 0 duplicate-owner net, bit 1 value
                              // counted by another rank (sharded halo mode)
  const int32_t* pin_inst;    // [n_pin] permuted
  const float4* off;          // [n_pin] permuted (rx_top, ry_top, rx_bot, ry_bot)
  const int32_t* slot;        // [n_pin] owner-sorted record slot of each permuted pin
  const double4* pos4;        // [n_inst] AoS centres
  double dz2, gamma, scale4, inv_gamma;
  const double* gamma_ptr;
  float4* out_f;              // [n_pin] (gx, gy, g_cut, FD) records by slot (fp32 mode)
  double* out_fd;             // unused
  double* out_d;              // [n_pin][4] float64 records by slot (fp64 mode)
  double* partials;
  unsigned int* counter;
  double* final6;
  const int* halt;
};

struct FusedGatherArgs {
  int n_obj, blocks;
  int obj0;                   // first object (the sharded halo mode sums its own slab only)
  const int32_t* obj_slot_ptr;
  const float4* in_f;         // fp32-mode records by slot
  const double* in_fd;
  const double* in_d;         // nullable: fp64-mode double4 records by slot
  double* out;                // [n_obj][4] (gx, gy, g_cut, FD)
  double* partials;
  unsigned int* counter;
  double* final_norms;
  const int* halt;
};

void launch_fused_net(const FusedNetArgs& a, bool f32, cudaStream_t s);

// multi-die 2D GP wirelength (p3d_gp2d.cu)
struct Gp2dWlArgs {
  int n_net, n_obj;
  const int32_t* net_ptr;      // [n_net+1] augmented CSR
  const int32_t* pin_obj;      // [n_pin]
  const uint8_t* pin_top;      // [n_pin] partial net (1: top)
  const double *pin_ox, *pin_oy;  // [n_pin] offsets frozen at the partition
  const int32_t* pin_slot;     // [n_pin] owner-sorted record slot
  const int32_t* obj_slot_ptr; // [n_obj+1]
  const double* pos;           // [2][n_obj]
  double gamma;
  const double* gamma_ptr;     // nullable: gamma from device memory (graph-captured loop)
  const int32_t* halt;         // nullable: return at once when set
  double* rec;                 // [n_pin][2] per-pin gradients by slot
  double* partials;            // [blocks]
  unsigned int* counter;
  double* value;               // 1 double: sum over segments of the WA spans
};
void launch_gp2d_wl(const Gp2dWlArgs& a, double* wl_grad, cudaStream_t s);
int gp2d_init(const p3d_gp2d_ctl& c, const double* pos0, cudaStream_t s);
int gp2d_step(const p3d_gp2d_ctl& c, cudaStream_t s);
int gp2d_project(const p3d_gp2d_ctl& c, const double* in, double* out, cudaStream_t s);
void launch_gp2d_layer_xy(int n, const int32_t* idx, const double* pos, int n_obj, double* x,
                          double* y, const int32_t* halt, cudaStream_t s);
void launch_gp2d_layer_force(int n, const int32_t* idx, const double* force, double* dens_grad,
                             const int32_t* halt, cudaStream_t s);

// post-GP steps (p3d_post.cu)
struct RebalanceArgs {
  int n;
  const double *area_top, *area_bot;     // [n] rotated w*h on each die
  const int32_t *order_top, *order_bot;  // [n] sorted by (is_macro, area on the die, index)
  uint8_t* delta;                        // [n] in/out: 1 top
  double cap_top, cap_bot;
  double* out;                           // [4]: status (0 ok, 1 unsatisfiable, 2 no convergence), moves, over_top, over_bot
};
void launch_rebalance(const RebalanceArgs& a, cudaStream_t s);
struct CheckArgs {
  int n_inst, n_net;
  const uint8_t* die;
  const int32_t* rot;
  const double *x, *y;
  const uint8_t* is_macro;
  const double *w_top, *h_top, *w_bot, *h_bot;
  const int32_t *net_ptr, *pin_inst;
  const uint8_t* hbt_ok;
  const double *hbt_x, *hbt_y;
  double die_w, die_h, row_top, row_bot, site_w, pitch, tol;
  uint8_t *inst_flags, *net_flags;
  double* box;    // [n_inst][4] x0, x1, y0, y1
  double* area;   // [2] per-die cell + macro area
  double* partials;  // [2 * kMaxBlocks]
  unsigned int* counter;
};
void launch_check(const CheckArgs& a, cudaStream_t s);
struct PairArgs {
  int n;
  const double* box;       // [n][4]
  const uint8_t* member;   // [n] 1: take part
  double bucket;
  int nbx, nby, mode;      // mode 0: overlap, 1: terminal spacing
  double min_cc, tol;
  int32_t *count, *start, *cursor, *list;
  int32_t* out;            // [cap_out][2] pairs (p < q)
  int32_t cap_out;
  int32_t* n_out;
};
void launch_pair_count(const PairArgs& a, cudaStream_t s);
void launch_pair_fill(const PairArgs& a, cudaStream_t s);
void launch_pair_test(const PairArgs& a, cudaStream_t s);

// small per-op kernels (p3d_ops.cu)
void launch_dynamic_size(int n, const double* wt, const double* ht, const double* wb,
                         const double* hb, const uint8_t* mac, const double* z, double dz,
                         double* w, double* h, cudaStream_t s);
void launch_axis_scan(int nx, int ny, int nz, int axis, bool reverse, double* a, cudaStream_t s);
void launch_overflow_d(long long n, const double* rho, double rho_t, double scale, double* scratch,
                       double* out, cudaStream_t s);
void launch_spans(int n, const int64_t* cnt, const double* min1, const double* max1,
                  const double* fmin, const double* fmax, double* top, double* bot, double* full,
                  cudaStream_t s);
void launch_bb_norms(long long n, const double* v, const double* vp, const double* g,
                     const double* ref, double* scratch, double* out, cudaStream_t s);
void launch_absmax(long long n, const double* g, double* scratch, double* out, cudaStream_t s);
void launch_axpy(long long n, const double* a, double sc, const double* b, const double* c,
                 double* out, cudaStream_t s);

// solution score (p3d_score.cu)
struct ScoreArgs {
  int n_net;
  const int32_t *net_ptr, *pin_inst;
  const double *ox_top, *oy_top, *ox_bot, *oy_bot;  // [n_pin]
  const double *w_top, *h_top, *w_bot, *h_bot;      // [n_inst] unrotated
  const uint8_t* die;
  const int32_t* rot;
  const double *x, *y;                               // lower-left corners
  const uint8_t* hbt_ok;                             // [n_net] net carries an HBT
  const double *hbt_x, *hbt_y;                       // [n_net] its lower-left corner
  double half, cost;
  double* partials;
  unsigned int* counter;
  int* n_bad;                                        // crossing / HBT mismatches
  double* out;                                       // hpwl, hbt count, raw score
};
void launch_score(const ScoreArgs& a, cudaStream_t s);
void fused_net_setup();
void launch_fused_gather(const FusedGatherArgs& a, cudaStream_t s);

int grid_blocks(int n, int threads, int cap);

// spatially ordered scatter (p3d_density.cu)
struct TileSort {
  int n_tiles, tiles_x, tiles_y, margin;
  int i0, ni, f0;    // object of local index k: k < ni ? i0 + k : f0 + (k - ni)
  int32_t* tile_of;  // [n_obj]
  int32_t* hist;     // [n_tiles] (kept zeroed between iterations)
  int32_t* start;    // [n_tiles + 1]
  int32_t* cursor;   // [n_tiles]
  int32_t* order;    // [n_obj] tile of each record, in tile order
  double* rec;       // [n_obj][6] charge records in tile order
  unsigned int* counter;  // last-block ticket of the histogram kernel
  // periodic re-sort: the counting sort runs when *it % every == 0 (or before
  // the first sort, *valid == 0); in between, the records are refreshed in the
  // last sort's order (perm[pos] = local object index).  rho is int64 fixed
  // point, so any record order gives the same map bit for bit.
  int32_t* perm;          // [n_obj] (null: sort every call)
  int32_t* valid;         // [1] set once perm holds a sort
  int32_t* decision;      // [1] this iteration's sort decision, written once by the
                          // histogram kernel's last block (place / scatter read it)
  const int32_t* it;      // the loop's iteration counter (null: sort every call)
  int every;
};
struct CloudGP;
void tiled_scatter_setup();
int tiled_scatter_tiles(const p3d_grid& g, int* tx, int* ty);
void launch_scatter_tiled(const CloudGP& cl, int n, int n_macro, const int32_t* macro_ids,
                          const p3d_grid& g, const TileSort& ts, int64_t* rho, const int* halt,
                          cudaStream_t s);

// K1
void launch_net_pos(const NetArgs& a, const double* x, const double* y, const double* z,
                    const double* off, double dz, cudaStream_t s);
void launch_net_direct(const NetArgs& a, const double* px, const double* py, const double* pz,
                       const uint8_t* top, bool planar, bool cut, bool fd, cudaStream_t s);
void launch_netboxes(const NetArgs& a, const double* c, const uint8_t* top, int64_t* cnt,
                     double* min1, double* min2, double* max1, double* max2, double* fmn,
                     double* fmx, double* bis, cudaStream_t s);
void launch_gather(const GatherArgs& a, cudaStream_t s);

// K3
struct SpecOvfl {  // overflow + re-zero fused into the first (fixed-point) pass
  int zero;
  long long rho_t_fx;
  double* partials;
  unsigned int* counter;
  double* out;
  double scale;    // 2^-40 * bin_vol / movable_volume
  // nullable (fast path only): the first pass adds its per-CTA excess to this
  // zeroed int64 total with one atomic each (no last-block reduction on the
  // pass's tail); the second pass converts it into *out and re-zeroes it
  unsigned long long* acc = nullptr;
};
int launch_spectral_ex(const p3d_grid* g, const double* rho, const int64_t* rho_fx,
                       const double* coef_in, double* coef_out, double* maps, double* scratch,
                       const int* halt, const SpecOvfl* ov, cudaStream_t s);
void spectral_setup();
bool spectral_fast_ok(const p3d_grid* g);
void spectral_fast_setup();
int launch_spectral_fast(const p3d_grid* g, const double* rho, const int64_t* rho_fx,
                         const double* coef_in, double* coef_out, double* maps, double* scratch,
                         const int* halt, const SpecOvfl* ov, cudaStream_t s);
void launch_scale_copy(const double* in, double* out, long long n, double s, cudaStream_t st);
int launch_spectral(const p3d_grid* g, const double* rho, const int64_t* rho_fx,
                    const double* coef_in, double* coef_out, double* maps, double* scratch,
                    const int* halt, cudaStream_t s);

}  // namespace p3d
