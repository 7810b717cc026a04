/*
 * p3d.h — C-ABI of libp3d.so, the B200 (sm_100a) global-placement hot path of
 * the arXiv 2403.09070 F2F 3D placer.
 *
 * Every entry point is stream-ordered and asynchronous: it enqueues kernels on
 * the given cudaStream_t (passed as void*) and returns.  All pointers are
 * DEVICE pointers unless noted; scalar results are written to device memory
 * (no implicit host synchronisation).  The library allocates nothing: the
 * caller owns every buffer (the Python host layer allocates them as torch
 * tensors).  Return value: P3D_OK or an error code; p3d_last_error() gives the
 * message.  Each declaration cites the reference routine it replaces
 * (paths relative to /root/reference/pkg/src/place3d).
 */
#ifndef P3D_H_
#define P3D_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define P3D_ABI_VERSION 1

#define P3D_OK 0
#define P3D_ERR_ARG 1          /* bad argument -> ValueError */
#define P3D_ERR_CUDA 2         /* launch / runtime failure -> RuntimeError */
#define P3D_ERR_UNSUPPORTED 3  /* size outside what this build handles */

/* ------------------------------------------------------------------------ */
/* library                                                                   */
/* ------------------------------------------------------------------------ */
int p3d_abi_version(void);
/* Copies the last error message (thread-local) into buf; returns its length. */
int p3d_last_error(char* buf, size_t n);
/* sizeof() of the structs below, so bindings can verify their mirrors. */
size_t p3d_sizeof_topology(void);
size_t p3d_sizeof_grid(void);
size_t p3d_sizeof_cloud(void);
size_t p3d_sizeof_gp(void);
size_t p3d_sizeof_loop_state(void);
/* Doubles the p3d_gp.partials buffer must hold (16 slots x 8 x 2048 blocks). */
size_t p3d_gp_partials_doubles(void);

/* ------------------------------------------------------------------------ */
/* netlist topology: CSR pins by net (wirelength.py:30-47 NetTopology)       */
/* ------------------------------------------------------------------------ */
typedef struct p3d_topology {
  int32_t n_net;
  int32_t n_pin;
  int32_t n_obj;             /* length of per-object outputs (gradient vector) */
  int32_t pad0;
  const int32_t* net_ptr;    /* [n_net+1] */
  const int32_t* pin_inst;   /* [n_pin] owner object of each pin */
  const uint8_t* net_dup;    /* [n_net] 1 if an owner has >= 2 pins in the net
                                (model.py:268-275 net_has_dup_inst) */
  const int32_t* net_order;  /* [n_net] processing order (nets grouped by
                                degree); NULL = identity */
  const int32_t* pin_slot;   /* [n_pin] position of the pin in owner-sorted
                                order; NULL = identity */
  const int32_t* obj_slot_ptr; /* [n_obj+1] slot range of each owner */
} p3d_topology;

/* Per-(net, die) first/second extrema with multiplicity on one axis
 * (wirelength.py:101-142 NetBoxes).  Outputs [n_net*2] (index 2*net+die) and
 * [n_net]; all nullable. */
int p3d_netboxes(const p3d_topology* t, const double* coord, const uint8_t* on_top,
                 int64_t* cnt, double* min1, double* min2, double* max1, double* max2,
                 double* full_min, double* full_max, double* spans_bistratal,
                 void* stream);

/* Smoothed bistratal planar WL and per-pin gradients, branch per net/axis from
 * the unsmoothed spans (wirelength.py:173-192 planar_objective).  value: one
 * device double.  gx/gy: [n_pin] (nullable).  scratch: zeroed device buffer of
 * >= 8 + 6*2048 doubles (reduction partials; left zeroed for reuse). */
int p3d_planar_objective_ex(const p3d_topology* t, const double* pin_x, const double* pin_y,
                            const uint8_t* on_top, double gamma, double* value, double* gx,
                            double* gy, double* scratch, void* stream);

/* WA z-span per net (wirelength.py:195-198 z_cut_penalty); scratch as above. */
int p3d_z_cut_penalty_ex(const p3d_topology* t, const double* pin_z, double gamma,
                         double* value, double* g, double* scratch, void* stream);

/* Incremental finite-difference depth gradient, accumulated per owner object
 * (wirelength.py:251-293 fd_z_gradient_incremental; exact O(|P|^2) path for
 * nets flagged in net_dup).  g: [n_obj]; requires net_dup, pin_slot and
 * obj_slot_ptr; pin_scratch: >= 4*n_pin + 4*n_obj doubles. */
int p3d_fd_z_gradient(const p3d_topology* t, const double* pin_x, const double* pin_y,
                      const uint8_t* on_top, double dz, double* g, double* pin_scratch,
                      void* stream);

/* Per-pin -> per-object ordered sums of up to 4 pin arrays laid out
 * [n_pin][4] in slot order (the np.bincount(pin_inst, w) of gp.py:307-309). */
int p3d_gather_pins(const p3d_topology* t, const double* pin4, double* obj4_soa,
                    void* stream);

/* dynamic_pin_coords (wirelength.py:308-322): pins from instance centres with
 * per-die rotated offsets.  off: [n_pin][4] (rx_top, ry_top, rx_bot, ry_bot). */
int p3d_pin_coords(const p3d_topology* t, const double* x, const double* y,
                   const double* z, const double* off, double dz, double* px,
                   double* py, double* pz, uint8_t* on_top, void* stream);

/* normalize_z_gradient (wirelength.py:296-305, Eq. 17); scratch: zeroed,
 * >= 8 + 3*1024 doubles. */
int p3d_normalize_z_gradient(int32_t n, const double* gx, const double* gy,
                             const double* gz_bist, const double* gz_hbt, double alpha,
                             double* out, double* scratch, void* stream);

/* ------------------------------------------------------------------------ */
/* density grid + spectral plan (density.py:26-55 DensityGrid)               */
/* ------------------------------------------------------------------------ */
typedef struct p3d_grid {
  int32_t nx, ny, nz, pad0;
  double dx, dy, dz, wb, hb, db, bin_vol;
  double fx_scale;           /* 2^40 / bin_vol (fixed-point density scale) */
  const double* omega[3];    /* [nx], [ny], [nz]: pi*k/d */
  const double* twiddle[3];  /* per axis: [n] (cos,sin)(-2 pi j/n), j < n/2; then, for
                                power-of-two n in [8,1024], the per-pass DIF table
                                W_{8s}^{qj} [pass][q-1][j] (density._pass_twiddles) */
  const double* phase[3];    /* per axis: [2n] (cos,sin)(pi k/(2n)) */
} p3d_grid;

/* Charges (density.py:58-83 ChargeCloud), SoA, length n. */
typedef struct p3d_cloud {
  int32_t n, n_macro;
  const double *x, *y, *z, *w, *h, *dep, *weight;
  const uint8_t* is_macro;
  const int32_t* macro_ids;  /* [n_macro] indices with is_macro set */
} p3d_cloud;

/* Fixed-point density accumulation (density.py:301-311 accumulate_density):
 * rho_fx [nx*ny*nz] int64 in units of 2^-40, ADDED into (caller zeroes). */
int p3d_accumulate_density(const p3d_grid* g, const p3d_cloud* c, int64_t* rho_fx,
                           void* stream);
/* rho = rho_fx * 2^-40 (exact). */
int p3d_fx_to_density(int64_t n, const int64_t* rho_fx, double* rho, void* stream);
/* overflow (density.py:612-617) from the fixed-point map; out: one double;
 * scratch: zeroed, >= 8 + 1024 doubles. */
int p3d_overflow_fx(const p3d_grid* g, const int64_t* rho_fx, double rho_t,
                    double movable_volume, double* out, double* scratch, void* stream);

/* Spectral Poisson solve + field (density.py:319-368).  rho: [B] float64.
 * coef (nullable): scipy-normalised dctn(rho, type=2).  maps (nullable):
 * [B][4] = (phi, Ex, Ey, Ez) interleaved.  scratch: >= 6*B doubles. */
int p3d_spectral(const p3d_grid* g, const double* rho, double* coef, double* maps,
                 double* scratch, void* stream);
/* The same from a given scipy-normalised coefficient array (electric_field). */
int p3d_spectral_from_coef(const p3d_grid* g, const double* coef, double* maps,
                           double* scratch, void* stream);
/* The loop's field solve straight from the int64 fixed-point map (rho_fx, 2^-40
 * per unit density): maps [B][4] (phi, Ex, Ey, Ez), the overflow of the map
 * against rho_t (density.py:612-617, movable volume mv) into ovfl_out[1], fused
 * into the first pass, and, with rezero, the map zeroed for the next
 * accumulation.  scratch: >= 6*B doubles; ovfl_scratch: >= 8 + 1024 doubles,
 * zeroed once (its ticket counter re-arms itself). */
int p3d_spectral_fx(const p3d_grid* g, int64_t* rho_fx, double* maps, double* scratch,
                    double rho_t, double mv, double* ovfl_out, double* ovfl_scratch, int rezero,
                    void* stream);

/* Overlap-weighted map means per charge (density.py:376-386, 489-609):
 * energy = sum q*phibar (one double), force[n][3] = -2 q Ebar (freeze: nullable
 * per-object mask zeroing the z component).  maps: [B][4].  scratch: zeroed,
 * >= 8 + n_macro + 1024 doubles. */
int p3d_density_gather(const p3d_grid* g, const p3d_cloud* c, const double* maps,
                       const uint8_t* freeze_z, double* energy, double* force,
                       double* scratch, void* stream);

/* density_energy_and_gradient (density.py:533-565): energy = sum q*phibar and
 * the exact gradient 2 w sum_b phi_b dvol/dc ([n][3]; cells: two face columns
 * per axis, density.py:389-441; macros: differentiated corner stamps against
 * the suffix-summed phi, density.py:444-502).  phi: [B]; freeze_z nullable.
 * scratch: >= B + 8 + 1024 doubles (suffix map, reduction partials), zeroed. */
int p3d_density_energy_gradient(const p3d_grid* g, const p3d_cloud* c, const double* phi,
                                const uint8_t* freeze_z, double* energy, double* grad,
                                double* scratch, void* stream);

/* Multi-die 2D GP wirelength (gp.py:586-600, _segment_wa wirelength.py:76-98
 * over the augmented pin list of gp.py:482-498): per (net, partial net)
 * weighted-average span on x and y; value = sum of all segment values (one
 * double); wl_grad [n_obj][2] = per-object owner sums of the per-pin
 * gradients in pin order.  pos [2][n_obj]; net_ptr/pin_* describe the
 * augmented CSR (pins sorted by net), pin_slot/obj_slot_ptr its owner-sorted
 * slots.  scratch: zeroed, >= 2*n_pin + 8 + 1024 doubles. */
int p3d_gp2d_wirelength(int32_t n_net, int32_t n_pin, int32_t n_obj, const int32_t* net_ptr,
                        const int32_t* pin_obj, const uint8_t* pin_top, const double* pin_ox,
                        const double* pin_oy, const int32_t* pin_slot,
                        const int32_t* obj_slot_ptr, const double* pos, double gamma,
                        double* value, double* wl_grad, double* scratch, void* stream);

/* p3d_gp2d_wirelength with the smoothing gamma read from device memory
 * (gamma_dev, the loop's schedule) and a halt flag (nullable: the loop's done
 * flag; the kernels return at once when set), for a graph-captured loop. */
int p3d_gp2d_wirelength_ex(int32_t n_net, int32_t n_pin, int32_t n_obj, const int32_t* net_ptr,
                           const int32_t* pin_obj, const uint8_t* pin_top, const double* pin_ox,
                           const double* pin_oy, const int32_t* pin_slot,
                           const int32_t* obj_slot_ptr, const double* pos,
                           const double* gamma_dev, const int32_t* halt, double* value,
                           double* wl_grad, double* scratch, void* stream);

/* Device-resident run_gp2d_multi loop (gp.py:640-681): the per-layer planar
 * fields and the wirelength are computed by the entry points above; the
 * per-layer lambda init (gp.py:643-649), the log row and stop test
 * (gp.py:650-656), the Eq. 19 preconditioning of the current and the
 * re-weighted previous gradient (gp.py:657-667), the Nesterov / BB step with
 * the 2D span clamp (gp.py:668-673, 178-227, 344-348) and the per-layer mu
 * update (gp.py:678-681) run in three kernels (p3d_gp2d_step) with all loop
 * control in p3d_gp2d_state: one iteration is graph-capturable, and nothing
 * is read back until the loop ends. */
typedef struct p3d_gp2d_state {
  int32_t it, done, diverged, converged;
  int32_t lam_set, step_set, iterations, pad0;
  double lam[3], prev_ovfl[3];
  double step, a, a_new, mom, dv2_next, gamma, final_overflow, gmax;
  uint32_t counters[8];
} p3d_gp2d_state;

typedef struct p3d_gp2d_ctl {
  int32_t n_obj, max_iters, n_hbt, nblk;
  const int32_t* layer;        /* [n_obj] 0 bottom, 1 top, 2 terminal layer */
  const double *size_w, *size_h;  /* [n_obj] planar sizes (gp.py:563-566) */
  const double* charge;        /* [n_obj] size_w * size_h * db (gp.py:640) */
  const uint8_t* is_macro;     /* [n_obj] */
  const double* degree;        /* [n_obj] (Eq. 19) */
  const double* gamma_tab;     /* [max_iters] */
  double die_w, die_h, stop_overflow, mu_min, mu_max, step_scale, min_step, pad1;
  double *u, *v;               /* [2][n_obj] */
  const double* wl_grad;       /* [n_obj][2] (p3d_gp2d_wirelength_ex) */
  const double* dens_grad;     /* [n_obj][2] (p3d_gp2d_layer_force) */
  const double* wl_value;      /* [1] */
  const double* ovfl;          /* [3] per-layer overflow (p3d_overflow_fx) */
  double *prev_wl, *prev_dens; /* [n_obj][2] raw gradients of the previous point */
  double* pre;                 /* [n_obj][2] the step's preconditioned gradient */
  double* partials;            /* >= 8 * nblk doubles */
  double* log;                 /* [max_iters][4]: it, WL value, #HBT, worst overflow */
  p3d_gp2d_state* st;
} p3d_gp2d_ctl;

size_t p3d_sizeof_gp2d_ctl(void);
size_t p3d_sizeof_gp2d_state(void);
/* state <- initial; u = v = project(pos0) (pos0 [2][n_obj]). */
int p3d_gp2d_init(const p3d_gp2d_ctl* c, const double* pos0, void* stream);
/* lambda init / log / stop, preconditioned BB step, projected advance. */
int p3d_gp2d_step(const p3d_gp2d_ctl* c, void* stream);
/* out = project(in) ([2][n_obj]; gp.py:571-575). */
int p3d_gp2d_project(const p3d_gp2d_ctl* c, const double* in, double* out, void* stream);
/* x[k] = pos[idx[k]], y[k] = pos[n_obj + idx[k]] (a layer's charge cloud). */
int p3d_gp2d_layer_xy(int32_t n, const int32_t* idx, const double* pos, int32_t n_obj, double* x,
                      double* y, const int32_t* halt, void* stream);
/* dens_grad[idx[k]] = force[k][0:2] (density_force of a layer, gp.py:624). */
int p3d_gp2d_layer_force(int32_t n, const int32_t* idx, const double* force, double* dens_grad,
                         const int32_t* halt, void* stream);

/* Solution score (evaluate_score, model.py:364-400): out[3] = (D2D HPWL, #HBT,
 * HPWL + hbt_cost * #HBT); n_bad[1] = nets whose crossing state disagrees with
 * their HBT (the reference's SolutionError cases).  Pins per net from
 * net_ptr/pin_inst; pin offsets from the instance centre per die; unrotated
 * instance sizes per die; die [n_inst] (1 top), rot [n_inst] quarter turns,
 * x/y lower-left corners; hbt_ok/hbt_x/hbt_y per net (lower-left corner).
 * scratch: zeroed, >= 8 + 2*1024 doubles. */
int p3d_score(int32_t n_net, const int32_t* net_ptr, const int32_t* pin_inst,
              const double* ox_top, const double* oy_top, const double* ox_bot,
              const double* oy_bot, const double* w_top, const double* h_top,
              const double* w_bot, const double* h_bot, const uint8_t* die, const int32_t* rot,
              const double* x, const double* y, const uint8_t* hbt_ok, const double* hbt_x,
              const double* hbt_y, double hbt_pitch, double hbt_cost, double* out, int32_t* n_bad,
              double* scratch, void* stream);

/* ------------------------------------------------------------------------ */
/* design input (host code)                                */
/* ------------------------------------------------------------------------ */
/* parse_design (model.py:423-571) + the Design checks (model.py:121-190) +
 * NetlistArrays (model.py:231-275) in one native pass over the text.  On a
 * malformed design returns P3D_ERR_ARG with the reference's message
 * (p3d_last_error: "line N: ..." for its ParseError cases, the DesignError
 * text otherwise).  handle: freed with p3d_parsed_free. */
int p3d_parse_design(const char* text, int64_t len, void** handle);
/* counts[5] = (n_inst, n_net, n_pin, inst-name bytes, net-name bytes);
 * scalars[9] = (die w, h, row height top, bottom, max util top, bottom,
 * HBT pitch, spacing, cost). */
int p3d_parsed_counts(const void* handle, int64_t* counts, double* scalars);
/* Fills the NetlistArrays fields (net_ptr [n_net+1], pin_* [n_pin], per-
 * instance sizes [n_inst]) and the names, each '\n'-terminated. */
int p3d_parsed_fill(const void* handle, uint8_t* is_macro, double* w_top, double* h_top,
                    double* w_bot, double* h_bot, int64_t* net_ptr, int64_t* pin_inst,
                    double* ox_top, double* oy_top, double* ox_bot, double* oy_bot,
                    char* inst_names, char* net_names);
void p3d_parsed_free(void* handle);

/* ------------------------------------------------------------------------ */
/* small per-op pieces of the operator API                                   */
/* ------------------------------------------------------------------------ */
/* dynamic_size (density.py:134-147): w, h [n] at depth z [n]. */
int p3d_dynamic_size(int32_t n, const double* w_top, const double* h_top, const double* w_bot,
                     const double* h_bot, const uint8_t* is_macro, const double* z, double dz,
                     double* w, double* h, void* stream);
/* prefix_sum_3d (reverse 0) / suffix_sum_3d (reverse 1) in place on a
 * C-ordered [nx][ny][nz] map (density.py:207-217): x, then y, then z. */
int p3d_prefix_sum_3d(int32_t nx, int32_t ny, int32_t nz, int32_t reverse, double* a,
                      void* stream);
/* overflow (density.py:612-617) of a float64 map [n]: out[1]; scratch: >= 8 +
 * 1024 doubles (counter zeroed once). */
int p3d_overflow(int64_t n, const double* rho, double rho_t, double bin_vol,
                 double movable_volume, double* out, double* scratch, void* stream);
/* NetBoxes.spans (wirelength.py:136-142): top, bottom, full [n_net]. */
int p3d_net_spans(int32_t n_net, const int64_t* cnt, const double* min1, const double* max1,
                  const double* full_min, const double* full_max, double* top, double* bot,
                  double* full, void* stream);
/* NesterovOptimizer.advance pieces (gp.py:198-226) over n doubles:
 * op 0: out[0] = |v - vp|^2, out[1] = |g - ref|^2;  op 1: out[0] = max |g|;
 * op 2: out = v + s * g (c null) or v + s * (g - c).  scratch: >= 8 + 2*2048. */
int p3d_nesterov_op(int32_t op, int64_t n, const double* v, const double* vp, const double* g,
                    const double* ref, double s, double* out, double* scratch, void* stream);

/* ------------------------------------------------------------------------ */
/* post-GP steps                                       */
/* ------------------------------------------------------------------------ */
/* rebalance_partition (legalize.py:464-499): moves instances off the die
 * that overshoots its utilisation cap more, cheapest first, until both caps
 * hold.  area_*: [n] rotated w*h per die; order_*: [n] all instances sorted
 * by (is_macro, area on that die, index); delta [n] (bit 0: 1 top) is
 * updated in place, bit 1 set on every instance that moved at least once.  out[4] = (status: 0 done, 1 caps unsatisfiable (LegalizationError),
 * 2 no convergence; moves; top overshoot; bottom overshoot).  One CTA. */
int p3d_rebalance(int32_t n, const double* area_top, const double* area_bot,
                  const int32_t* order_top, const int32_t* order_bot, uint8_t* delta,
                  double cap_top, double cap_bot, double* out, void* stream);

/* check_solution (check.py:74-152), per-object part: inst_flags [n_inst]
 * (bit 0 rotated cell, 1 out of the die, 2 off the row grid, 3 off the site
 * grid), box [n_inst][4] (x0, x1, y0, y1 of the rotated outline), area[2]
 * (per die), net_flags [n_net] (bit 0 crossing net without terminal, 1
 * single-die net with one, 2 terminal out of the die).  x, y: lower-left
 * corners; w/h_*: unrotated outline per die; hbt_*: per net.
 * scratch: >= 2*2048 + 8 doubles (counter zeroed once). */
int p3d_check_objects(int32_t n_inst, int32_t n_net, const uint8_t* die, const int32_t* rot,
                      const double* x, const double* y, const uint8_t* is_macro,
                      const double* w_top, const double* h_top, const double* w_bot,
                      const double* h_bot, const int32_t* net_ptr, const int32_t* pin_inst,
                      const uint8_t* hbt_ok, const double* hbt_x, const double* hbt_y,
                      double die_w, double die_h, double row_top, double row_bot, double site_w,
                      double pitch, double tol, uint8_t* inst_flags, uint8_t* net_flags,
                      double* box, double* area, double* scratch, void* stream);
/* Pair search over boxes [n][4] (members only) on an nbx x nby grid of
 * `bucket`-sized buckets (check.py:47-71): phase 0 counts entries per bucket
 * into count [nbx*nby] (zeroed); phase 1 fills list [sum count] from start
 * [nbx*nby + 1] (exclusive scan of count; cursor = a copy of start); phase 2
 * tests every pair of every bucket (mode 0: outlines overlap by more than
 * 1e-9; mode 1: terminal boxes overlap and max(|dx|, |dy|) < min_cc - tol)
 * and writes each hit once as (p, q), p < q, into out [cap][2]; n_out[1]
 * counts all hits (may exceed cap). */
int p3d_pair_search(int32_t phase, int32_t n, const double* box, const uint8_t* member,
                    double bucket, int32_t nbx, int32_t nby, int32_t mode, double min_cc,
                    double tol, int32_t* count, int32_t* start, int32_t* cursor, int32_t* list,
                    int32_t* out, int32_t cap, int32_t* n_out, void* stream);

/* ------------------------------------------------------------------------ */
/* optimiser pieces (gp.py:142-147, 178-227, 280-294)                        */
/* ------------------------------------------------------------------------ */
/* precondition: out[n][3] = g / max(1, lam*q + macro*deg); div[n]. */
int p3d_precondition(int32_t n, const double* g, double lam, const double* q,
                     const double* deg, const uint8_t* macro, double* out, double* div,
                     void* stream);

/* ------------------------------------------------------------------------ */
/* the fused device-resident GP loop (gp.py:359-455 run_gp3d)                */
/* ------------------------------------------------------------------------ */
typedef struct p3d_loop_state {
  /* control */
  int32_t it, done, diverged, lam_set;
  int32_t step_set, stop_now, best_flag, rise;
  int32_t nonfinite, converged, eval_only, pad0;
  /* schedule / optimiser scalars */
  double lam, a, step, a_new, mom;
  double prev_ovfl, prev_value, last_mu, best0, best1;
  /* results of the current evaluation */
  double wl_x, wl_y, cut, exact, ncross;
  double norm_x, norm_y, norm_zb, gz_scale;
  double energy, ovfl, value, wl_value, l1_wl, l1_dens;
  double gamma, lam_eval;
  double dv2, dg2, gmax;
  double dv2_next;             /* |v_new - v|^2 of the last advance (BB numerator) */
  /* GpInfo */
  int32_t iterations, hbt_count;
  double final_overflow, wirelength;
  uint32_t counters[16];
} p3d_loop_state;

typedef struct p3d_gp {
  int32_t n_inst, n_fill, n_obj, n_macro;
  int32_t max_iters, divergence_window, nblk_obj, nblk_net;
  int32_t wl_f32;              /* 1: WA sums in fp32 on anchored differences */
  int32_t nblk_dens;           /* K4 CTAs (besides one per macro) */
  p3d_topology topo;           /* n_obj = n_inst here */
  /* degree-bucketed, transposed pin layout of the fused K1 (built by the host) */
  int32_t f_n_tasks, f_n_generic;
  const int32_t* f_generic_nets; /* [f_n_generic] permuted indices of nets with degree
                                    outside [2, 6] (per-thread generic path) */
  const int32_t* f_tasks;      /* [f_n_tasks][4] warp tasks (pin base, bucket size, j0, deg) */
  const int32_t* f_task_t0;    /* [f_n_tasks] permuted index of the bucket's first net */
  const int32_t *f_net_base, *f_net_deg, *f_net_stride;  /* [n_net] permuted nets */
  const uint8_t* f_net_dup;                             /* [n_net] */
  const int32_t* f_pin_inst;                            /* [n_pin] permuted pins */
  const float* f_pin_off;                               /* [n_pin][4] */
  const int32_t* f_pin_slot;   /* [n_pin] owner-sorted record slot of each permuted pin */
  p3d_grid grid;
  /* per-object constants */
  const double* pin_off;       /* [n_pin][4] rotated (rx_top, ry_top, rx_bot, ry_bot) */
  const double *w_top, *h_top, *w_bot, *h_bot;  /* [n_inst], rotated dims */
  const uint8_t* is_macro;     /* [n_inst] */
  const double* degree;        /* [n_inst] pin counts (Eq. 19) */
  const double *fill_w, *fill_h, *fill_z;       /* [n_fill] */
  const int32_t* macro_ids;    /* [n_macro] */
  const double* gamma_tab;     /* [max_iters] gamma schedule (gp.py:171-175) */
  /* scalars */
  double alpha, target_density, movable_volume, stop_overflow;
  double mu_min, mu_max, gamma0, gamma1, min_step, step_scale;
  int64_t rho_t_fx;
  /* state, [3][n_obj] SoA unless noted */
  double *u, *v;
  double *v_prev;              /* unused since the step reduces |v_new - v|^2 itself
                                  (kept for ABI stability; may be null) */
  double *best;
  double *wl_grad, *dens_grad, *pre, *prev_wl, *prev_dens;
  double* prev_q;              /* [n_obj] */
  double* pin_out;             /* [n_pin][4] slot order (exact mode) */
  float* pin_out_f;            /* [n_pin][4] slot order (gx, gy, g_cut, 0) */
  double* pin_out_fd;          /* [n_pin] slot order FD depth term */
  double* pos4;                /* [n_inst][4] AoS copy of v (x, y, z, 0) */
  double* inst_g;              /* [n_inst][4] gx, gy, gz_hbt, gz_bist (sharded: rows
                                  padded to shard_size equal slabs) */
  int64_t* rho_fx;             /* [B] */
  /* spatial tile sort of the objects for the privatised scatter (K2) */
  int32_t ts_n_tiles, ts_tiles_x, ts_tiles_y;
  int32_t ts_margin;           /* bins an object footprint can reach past its centre tile */
  int32_t *ts_tile_of, *ts_hist, *ts_start, *ts_cursor, *ts_order;  /* [O], [T], [T+1], [T], [2O+2]:
                                  ts_order = tile of each record in tile order, then the
                                  sort permutation [O], a permutation-valid flag and the
                                  iteration's sort decision (the sort reruns every
                                  P3D_RESORT_EVERY iterations) */
  double* ts_rec;              /* [O][6] charge records (x, y, z, w, h, weight) in tile order */
  double* rho;                 /* [B] */
  double* spec_scratch;        /* [6*B] */
  double* maps;                /* [B][4] */
  double* partials;            /* [16][8 * 2048] = p3d_gp_partials_doubles() doubles:
                                  16 slots of per-block partial sums (8 per block, up
                                  to 2048 blocks per launch) */
  p3d_loop_state* st;
  double* log;                 /* [max_iters][4]: it, exact WL, crossings, overflow */
  double* ovfl_hist;           /* [max_iters] */
  /* sharded loop (p3d_gp_shard_stage): this rank owns the instance
   * range [sh_i0, sh_i1) and the filler range [sh_f0, sh_f1) (object indices)
   * and the K1 warp tasks w with w % shard_size == shard_rank; n_macro /
   * macro_ids then list its own macros.  shard_size = 0 selects the fused
   * single-GPU loop (p3d_gp_iterate; sh_i0 = 0, sh_i1 = n_inst, sh_f0 = n_inst,
   * sh_f1 = n_obj); shard_size >= 1 the staged protocol (world size). */
  int32_t shard_rank, shard_size;
  int32_t sh_i0, sh_i1, sh_f0, sh_f1;
  double* shard_tot;           /* [32] per-rank totals the host all-reduces between
                                  stages: [0,6) net totals, [8,14) density totals,
                                  [16] max |g| (iteration 0), [20,23) L1 norms */
  int32_t overlap;             /* 1: the wirelength branch (K1, K1b) runs on a side
                                  stream concurrently with the density branch (K2,
                                  K3), joined before K4 (fused loop) */
  int32_t shard_halo;          /* sharded loop only: 1 = halo mode (each rank runs its own
                                  task list: every net touching its instance slab, and
                                  counts the value of the nets whose f_net_dup bit 1 is
                                  clear; owner sums over its own slab only, no owner-sum
                                  exchange); 0 = tasks dealt round-robin + reduce-scatter */
} p3d_gp;

/* Stages of one sharded GP iteration.  The host runs them in this order with
 * the collectives in brackets (sum unless noted):
 *   NET, GATHER, [reduce-scatter inst_g slabs], NORMS, [shard_tot[20:23]],
 *   NORMS_FINAL, SCATTER, [rho_fx (int64, exact)], SPECTRAL,
 *   DENS, [shard_tot[0:16]], CONTROL, STEP0, [shard_tot[16], max],
 *   STEP0_CONTROL, ADVANCE, [st->dv2_next], [all-gather of pos4 slabs]. */
enum {
  P3D_SH_NET = 0,
  P3D_SH_GATHER = 1,
  P3D_SH_NORMS = 2,
  P3D_SH_SCATTER = 3,
  P3D_SH_SPECTRAL = 4,
  P3D_SH_DENS = 5,
  P3D_SH_CONTROL = 6,
  P3D_SH_STEP0 = 7,
  P3D_SH_STEP0_CONTROL = 8,
  P3D_SH_ADVANCE = 9,
  P3D_SH_NORMS_FINAL = 10,
  P3D_SH_N_STAGES = 11
};

/* Reset the loop state (lambda unset, a = 1, iteration 0) and project u = v =
 * P(pos0) (gp.py:188-196); pos0 [3][n_obj] may alias u. */
int p3d_gp_init(const p3d_gp* gp, const double* pos0, void* stream);
/* One full GP iteration (gp.py:386-444) with all control on the device;
 * a no-op once st->done is set.  Capturable in a CUDA graph. */
int p3d_gp_iterate(const p3d_gp* gp, void* stream);
/* p3d_gp_iterate without the iteration-0 initial-step kernel (gp.py:198-202),
 * for every iteration after the first: that kernel is a no-op once the first
 * step is set, and leaving it out removes a dependency hop from the step's
 * tail.  Call it only after one p3d_gp_iterate since the last p3d_gp_init:
 * called at iteration 0 (no initial step yet) the step kernel ends the loop
 * with st->diverged and st->done set instead of advancing. */
int p3d_gp_iterate_steady(const p3d_gp* gp, void* stream);
/* Gp3dProblem.evaluate (gp.py:296-341) at gp->v with the given lambda and
 * gamma, filling wl_grad, dens_grad, rho_fx -> maps and the st result fields
 * (no optimiser step, loop control untouched). */
int p3d_gp_evaluate(const p3d_gp* gp, double lam, double gamma, void* stream);
/* p3d_gp_iterate with a CUDA event between the stages K1 (net), K1b (owner
 * gather), K2 (scatter), K3 (spectral), K4 (density gather + assembly),
 * K5a (precondition/BB), K5b (advance); stage_ms: HOST float[7].  Blocks until
 * the iteration finishes.  Not capturable (benchmark attribution only). */
int p3d_gp_iterate_profiled(const p3d_gp* gp, void* stream, float* stage_ms);
/* p3d_gp_iterate with library-owned stage events recorded as external
 * event nodes (capturable); p3d_gp_stage_times then waits for the last event
 * and returns the 7 stage durations (ms, HOST float[7]) of the most recent
 * marked iteration (e.g. a replayed graph). */
int p3d_gp_iterate_marked(const p3d_gp* gp, void* stream);
/* The overlapped (production) iteration with event-record nodes at its branch
 * points (graph-capturable, descriptors with overlap set); then
 * p3d_gp_overlap_times(t[7]): ms from the fork to the end of K1, K1b (WL
 * branch), K2, K3 (density branch), K4, K5a, K5b. */
int p3d_gp_iterate_marked_overlap(const p3d_gp* gp, void* stream);
int p3d_gp_overlap_times(float* t);
int p3d_gp_stage_times(float* stage_ms);
/* Number of kernels one p3d_gp_iterate enqueues (>0), or -1 on bad input. */
int p3d_gp_kernels_per_iteration(const p3d_gp* gp);
/* The loop's K2 alone (spatially sorted, shared-memory privatised scatter;
 * accumulate_density, density.py:301-311) at gp->v: the int64 fixed-point map
 * is written to out [B] and gp->rho_fx is left zeroed. */
int p3d_gp_density_fx(const p3d_gp* gp, int64_t* out, void* stream);
/* One stage of a sharded GP iteration (see P3D_SH_*); a no-op once st->done. */
int p3d_gp_shard_stage(const p3d_gp* gp, int stage, void* stream);
/* Gp3dProblem.project (gp.py:280-294): out = P(in), [3][n_obj]. */
int p3d_gp_project(const p3d_gp* gp, const double* in, double* out, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* P3D_H_ */
