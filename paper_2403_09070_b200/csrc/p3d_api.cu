// extern "C" entry points of libp3d.so (declared in include/p3d.h).
// Argument validation, error strings, and dispatch to the kernel launchers.
#include <stdarg.h>
#include <stdio.h>
#include <string.h>

#include "p3d_common.cuh"
#include "p3d_geom.cuh"
#include "p3d_internal.cuh"

namespace p3d {

static thread_local char g_err[512] = {0};

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

int check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("%s: %s", what, cudaGetErrorString(e));
    return P3D_ERR_CUDA;
  }
  return P3D_OK;
}

template <class Cloud>
void launch_scatter(const Cloud& cl, int n, int n_macro, const int32_t* macro_ids,
                    const p3d_grid& g, int64_t* rho, const int* halt, cudaStream_t s);
void launch_energy_grad(const p3d_cloud& c, const p3d_grid& g, const double* phi,
                        const uint8_t* freeze, double* energy, double* grad, double* scratch,
                        cudaStream_t s);
void launch_gather_op(const p3d_cloud& c, const p3d_grid& g, const double* maps,
                      const uint8_t* freeze, double* energy, double* force, double* scratch,
                      cudaStream_t s);
void launch_fx_to_density(long long n, const int64_t* in, double* out, cudaStream_t s);
void launch_overflow(long long n, const int64_t* rho, long long t, double scale, double* scratch,
                     double* out, cudaStream_t s);
void launch_precondition(int n, const double* g, double lam, const double* q, const double* deg,
                         const uint8_t* macro, double* out, double* div, cudaStream_t s);
void launch_pin_coords(int n_pin, const int32_t* pin_inst, const double* x, const double* y,
                       const double* z, const double* off, double dz, double* px, double* py,
                       double* pz, uint8_t* top, cudaStream_t s);
void launch_normalize(int n, const double* gx, const double* gy, const double* gzb,
                      const double* gzh, double alpha, double* out, double* scratch,
                      cudaStream_t s);
int gp_iterate(const p3d_gp& gp, cudaStream_t s, bool steady = false);
int gp_iterate_marked_overlap(const p3d_gp& gp, cudaStream_t s);
int gp_overlap_times(float* t);
int gp_evaluate(const p3d_gp& gp, double lam, double gamma, cudaStream_t s);
int gp_init(const p3d_gp& gp, const double* pos0, cudaStream_t s);
int gp_project(const p3d_gp& gp, const double* in, double* out, cudaStream_t s);
int gp_density_fx(const p3d_gp& gp, int64_t* out, cudaStream_t s);
int gp_shard_stage(const p3d_gp& gp, int stage, cudaStream_t s);
int gp_iterate_profiled(const p3d_gp& gp, cudaStream_t s, float* ms);
int gp_kernels_per_iteration(const p3d_gp& gp);
int gp_iterate_marked(const p3d_gp& gp, cudaStream_t s);
int gp_stage_times(float* ms);

static NetArgs net_args(const p3d_topology* t) {
  NetArgs a{};
  a.n_net = t->n_net;
  a.blocks = grid_blocks(t->n_net, 256, kMaxBlocks);
  a.net_ptr = t->net_ptr;
  a.pin_inst = t->pin_inst;
  a.net_order = t->net_order;
  a.net_dup = t->net_dup;
  a.pin_slot = nullptr;
  return a;
}

static bool bad_topo(const p3d_topology* t) {
  if (!t || t->n_net < 0 || t->n_pin < 0 || !t->net_ptr || (t->n_pin > 0 && !t->pin_inst)) {
    set_error("invalid topology");
    return true;
  }
  return false;
}

static bool bad_grid(const p3d_grid* g) {
  if (!g || g->nx <= 0 || g->ny <= 0 || g->nz <= 0 || !(g->bin_vol > 0)) {
    set_error("invalid grid");
    return true;
  }
  for (int k = 0; k < 3; ++k)
    if (!g->omega[k] || !g->twiddle[k] || !g->phase[k]) {
      set_error("grid tables missing");
      return true;
    }
  return false;
}

}  // namespace p3d

using namespace p3d;

#define STREAM(s) reinterpret_cast<cudaStream_t>(s)

extern "C" {

int p3d_abi_version(void) { return P3D_ABI_VERSION; }

int p3d_last_error(char* buf, size_t n) {
  size_t l = strlen(g_err);
  if (buf && n) {
    size_t c = l < n - 1 ? l : n - 1;
    memcpy(buf, g_err, c);
    buf[c] = 0;
  }
  return (int)l;
}

size_t p3d_sizeof_topology(void) { return sizeof(p3d_topology); }
size_t p3d_sizeof_grid(void) { return sizeof(p3d_grid); }
size_t p3d_sizeof_cloud(void) { return sizeof(p3d_cloud); }
size_t p3d_sizeof_gp(void) { return sizeof(p3d_gp); }
size_t p3d_sizeof_loop_state(void) { return sizeof(p3d_loop_state); }
size_t p3d_gp_partials_doubles(void) { return (size_t)16 * kPartialStride; }

int p3d_netboxes(const p3d_topology* t, const double* coord, const uint8_t* on_top, int64_t* cnt,
                 double* min1, double* min2, double* max1, double* max2, double* full_min,
                 double* full_max, double* spans, void* stream) {
  if (bad_topo(t) || !coord || !on_top) return P3D_ERR_ARG;
  if (t->n_net == 0) return P3D_OK;
  NetArgs a = net_args(t);
  launch_netboxes(a, coord, on_top, cnt, min1, min2, max1, max2, full_min, full_max, spans,
                  STREAM(stream));
  return check_launch("netboxes");
}

// scratch for reductions: caller-provided value buffer must hold >= 1 double;
// the per-op WL reductions use a small scratch carved from `value`'s neighbour
// arrays: value[0] result, value[1..] are NOT used.  Partials live in gx/gy-free
// scratch allocated by the caller through p3d_planar_objective_ex.
static int planar_like(const p3d_topology* t, const double* px, const double* py,
                       const double* pz, const uint8_t* top, double gamma, double* value,
                       int value_mode, double* gx, double* gy, double* gc, bool planar, bool cut,
                       double* scratch, cudaStream_t s) {
  NetArgs a = net_args(t);
  a.gamma = gamma;
  a.want_pins = (gx || gy || gc) ? 1 : 0;
  a.gx = gx;
  a.gy = gy;
  a.gc = gc;
  a.value_mode = value_mode;
  a.value_out = value;
  a.counter = reinterpret_cast<unsigned int*>(scratch);
  a.final6 = scratch + 2;
  a.partials = scratch + 8;
  launch_net_direct(a, px, py, pz, top, planar, cut, false, s);
  return check_launch(planar ? "planar_objective" : "z_cut_penalty");
}

int p3d_planar_objective_ex(const p3d_topology* t, const double* pin_x, const double* pin_y,
                            const uint8_t* on_top, double gamma, double* value, double* gx,
                            double* gy, double* scratch, void* stream) {
  if (bad_topo(t) || !pin_x || !pin_y || !on_top || !value || !scratch) {
    if (!g_err[0]) set_error("planar_objective: null argument");
    return P3D_ERR_ARG;
  }
  if (!(gamma > 0)) { set_error("gamma must be positive"); return P3D_ERR_ARG; }
  return planar_like(t, pin_x, pin_y, nullptr, on_top, gamma, value, 0, gx, gy, nullptr, true,
                     false, scratch, STREAM(stream));
}

int p3d_z_cut_penalty_ex(const p3d_topology* t, const double* pin_z, double gamma, double* value,
                         double* g, double* scratch, void* stream) {
  if (bad_topo(t) || !pin_z || !value || !scratch) { set_error("z_cut_penalty: null argument"); return P3D_ERR_ARG; }
  if (!(gamma > 0)) { set_error("gamma must be positive"); return P3D_ERR_ARG; }
  return planar_like(t, nullptr, nullptr, pin_z, nullptr, gamma, value, 1, nullptr, nullptr, g,
                     false, true, scratch, STREAM(stream));
}

int p3d_fd_z_gradient(const p3d_topology* t, const double* pin_x, const double* pin_y,
                      const uint8_t* on_top, double dz, double* g, double* pin_scratch,
                      void* stream) {
  if (bad_topo(t) || !pin_x || !pin_y || !on_top || !g || !pin_scratch || !t->pin_slot ||
      !t->obj_slot_ptr || !t->net_dup) {
    set_error("fd_z_gradient: null argument (needs pin_slot, obj_slot_ptr, net_dup)");
    return P3D_ERR_ARG;
  }
  cudaStream_t s = STREAM(stream);
  NetArgs a = net_args(t);
  a.gamma = 1.0;
  a.scale4 = 4.0 / dz;
  a.want_pins = 1;
  a.pin_slot = t->pin_slot;
  // the FD term lands in column 3 of a [n_pin][4] slot array
  a.out4 = pin_scratch;
  cudaMemsetAsync(pin_scratch, 0, sizeof(double) * 4 * (size_t)t->n_pin, s);
  if (t->n_net > 0) launch_net_direct(a, pin_x, pin_y, nullptr, on_top, false, false, true, s);
  GatherArgs ga{};
  ga.n_obj = t->n_obj;
  ga.blocks = grid_blocks(t->n_obj, 256, kMaxBlocks);
  ga.obj_slot_ptr = t->obj_slot_ptr;
  ga.pin4 = pin_scratch;
  // gather all four columns into pin_scratch's tail? keep simple: columns to a
  // caller-visible [4][n_obj] area placed after the pin array
  double* out4 = pin_scratch + 4 * (size_t)t->n_pin;
  ga.out = out4;
  launch_gather(ga, s);
  cudaMemcpyAsync(g, out4 + 3 * (size_t)t->n_obj, sizeof(double) * t->n_obj,
                  cudaMemcpyDeviceToDevice, s);
  return check_launch("fd_z_gradient");
}

int p3d_gather_pins(const p3d_topology* t, const double* pin4, double* obj4, void* stream) {
  if (bad_topo(t) || !pin4 || !obj4 || !t->obj_slot_ptr) { set_error("gather_pins: null argument"); return P3D_ERR_ARG; }
  GatherArgs ga{};
  ga.n_obj = t->n_obj;
  ga.blocks = grid_blocks(t->n_obj, 256, kMaxBlocks);
  ga.obj_slot_ptr = t->obj_slot_ptr;
  ga.pin4 = pin4;
  ga.out = obj4;
  launch_gather(ga, STREAM(stream));
  return check_launch("gather_pins");
}

int p3d_pin_coords(const p3d_topology* t, const double* x, const double* y, const double* z,
                   const double* off, double dz, double* px, double* py, double* pz,
                   uint8_t* on_top, void* stream) {
  if (bad_topo(t) || !x || !y || !z || !off) { set_error("pin_coords: null argument"); return P3D_ERR_ARG; }
  if (t->n_pin == 0) return P3D_OK;
  launch_pin_coords(t->n_pin, t->pin_inst, x, y, z, off, dz, px, py, pz, on_top, STREAM(stream));
  return check_launch("pin_coords");
}

int p3d_normalize_z_gradient(int32_t n, const double* gx, const double* gy, const double* gzb,
                             const double* gzh, double alpha, double* out, double* scratch,
                             void* stream) {
  if (n < 0 || !gx || !gy || !gzb || !gzh || !out || !scratch) { set_error("normalize: null argument"); return P3D_ERR_ARG; }
  if (n == 0) return P3D_OK;
  launch_normalize(n, gx, gy, gzb, gzh, alpha, out, scratch, STREAM(stream));
  return check_launch("normalize_z_gradient");
}

int p3d_accumulate_density(const p3d_grid* g, const p3d_cloud* c, int64_t* rho_fx,
                           void* stream) {
  if (bad_grid(g) || !c || !rho_fx || c->n < 0) { if (!g_err[0]) set_error("accumulate: bad args"); return P3D_ERR_ARG; }
  if (c->n == 0) return P3D_OK;
  if (c->n_macro > 0 && !c->macro_ids) { set_error("macro_ids missing"); return P3D_ERR_ARG; }
  CloudArrays cl;
  cl.c = *c;
  launch_scatter(cl, c->n, c->n_macro, c->macro_ids, *g, rho_fx, nullptr, STREAM(stream));
  return check_launch("accumulate_density");
}

int p3d_fx_to_density(int64_t n, const int64_t* rho_fx, double* rho, void* stream) {
  if (n < 0 || !rho_fx || !rho) { set_error("fx_to_density: bad args"); return P3D_ERR_ARG; }
  if (n == 0) return P3D_OK;
  launch_fx_to_density(n, rho_fx, rho, STREAM(stream));
  return check_launch("fx_to_density");
}

int p3d_overflow_fx(const p3d_grid* g, const int64_t* rho_fx, double rho_t, double mv, double* out,
                    double* scratch, void* stream) {
  if (bad_grid(g) || !rho_fx || !out || !scratch) { if (!g_err[0]) set_error("overflow: bad args"); return P3D_ERR_ARG; }
  const long long n = (long long)g->nx * g->ny * g->nz;
  const long long t = __builtin_llrint(rho_t * 1099511627776.0);
  const double scale = mv > 0 ? 9.094947017729282379150390625e-13 * g->bin_vol / mv : 0.0;
  launch_overflow(n, rho_fx, t, scale, scratch, out, STREAM(stream));
  return check_launch("overflow");
}

int p3d_spectral(const p3d_grid* g, const double* rho, double* coef, double* maps,
                 double* scratch, void* stream) {
  if (bad_grid(g) || !rho || !scratch) { if (!g_err[0]) set_error("spectral: bad args"); return P3D_ERR_ARG; }
  return launch_spectral_ex(g, rho, nullptr, nullptr, coef, maps, scratch, nullptr, nullptr,
                            STREAM(stream));
}

int p3d_spectral_fx(const p3d_grid* g, int64_t* rho_fx, double* maps, double* scratch,
                    double rho_t, double mv, double* ovfl_out, double* ovfl_scratch, int rezero,
                    void* stream) {
  if (bad_grid(g) || !rho_fx || !maps || !scratch || !ovfl_out || !ovfl_scratch) {
    if (!g_err[0]) set_error("spectral_fx: bad args");
    return P3D_ERR_ARG;
  }
  SpecOvfl ov;
  ov.zero = rezero ? 1 : 0;
  ov.rho_t_fx = __builtin_llrint(rho_t * 1099511627776.0);
  ov.partials = ovfl_scratch + 8;
  ov.counter = reinterpret_cast<unsigned int*>(ovfl_scratch);
  ov.out = ovfl_out;
  ov.scale = mv > 0 ? 9.094947017729282379150390625e-13 * g->bin_vol / mv : 0.0;
  return launch_spectral_ex(g, nullptr, rho_fx, nullptr, nullptr, maps, scratch, nullptr, &ov,
                            STREAM(stream));
}

int p3d_spectral_from_coef(const p3d_grid* g, const double* coef, double* maps, double* scratch,
                           void* stream) {
  if (bad_grid(g) || !coef || !maps || !scratch) { if (!g_err[0]) set_error("spectral: bad args"); return P3D_ERR_ARG; }
  return launch_spectral_ex(g, nullptr, nullptr, coef, nullptr, maps, scratch, nullptr, nullptr,
                            STREAM(stream));
}

int p3d_density_gather(const p3d_grid* g, const p3d_cloud* c, const double* maps,
                       const uint8_t* freeze_z, double* energy, double* force, double* scratch,
                       void* stream) {
  if (bad_grid(g) || !c || !maps || !energy || !force || !scratch) { if (!g_err[0]) set_error("density_gather: bad args"); return P3D_ERR_ARG; }
  if (c->n_macro > 0 && !c->macro_ids) { set_error("macro_ids missing"); return P3D_ERR_ARG; }
  launch_gather_op(*c, *g, maps, freeze_z, energy, force, scratch, STREAM(stream));
  return check_launch("density_gather");
}

int p3d_density_energy_gradient(const p3d_grid* g, const p3d_cloud* c, const double* phi,
                                const uint8_t* freeze_z, double* energy, double* grad,
                                double* scratch, void* stream) {
  if (bad_grid(g) || !c || !phi || !energy || !grad || !scratch) { if (!g_err[0]) set_error("density_energy_gradient: bad args"); return P3D_ERR_ARG; }
  if (c->n == 0) return P3D_OK;
  launch_energy_grad(*c, *g, phi, freeze_z, energy, grad, scratch, STREAM(stream));
  return check_launch("density_energy_gradient");
}

int p3d_gp2d_wirelength(int32_t n_net, int32_t n_pin, int32_t n_obj, const int32_t* net_ptr,
                        const int32_t* pin_obj, const uint8_t* pin_top, const double* pin_ox,
                        const double* pin_oy, const int32_t* pin_slot,
                        const int32_t* obj_slot_ptr, const double* pos, double gamma,
                        double* value, double* wl_grad, double* scratch, void* stream) {
  if (n_net < 0 || n_pin < 0 || n_obj < 0 || !net_ptr || !pos || !value || !wl_grad || !scratch ||
      (n_pin > 0 && (!pin_obj || !pin_top || !pin_ox || !pin_oy || !pin_slot)) || !obj_slot_ptr ||
      !(gamma > 0)) {
    set_error("gp2d_wirelength: bad args");
    return P3D_ERR_ARG;
  }
  Gp2dWlArgs a{};
  a.n_net = n_net; a.n_obj = n_obj;
  a.net_ptr = net_ptr; a.pin_obj = pin_obj; a.pin_top = pin_top;
  a.pin_ox = pin_ox; a.pin_oy = pin_oy; a.pin_slot = pin_slot; a.obj_slot_ptr = obj_slot_ptr;
  a.pos = pos; a.gamma = gamma;
  a.gamma_ptr = nullptr; a.halt = nullptr;
  a.rec = scratch;
  a.counter = reinterpret_cast<unsigned int*>(scratch + 2 * (long long)n_pin);
  a.partials = scratch + 2 * (long long)n_pin + 8;
  a.value = value;
  launch_gp2d_wl(a, wl_grad, STREAM(stream));
  return check_launch("gp2d_wirelength");
}

int p3d_score(int32_t n_net, const int32_t* net_ptr, const int32_t* pin_inst,
              const double* ox_top, const double* oy_top, const double* ox_bot,
              const double* oy_bot, const double* w_top, const double* h_top,
              const double* w_bot, const double* h_bot, const uint8_t* die, const int32_t* rot,
              const double* x, const double* y, const uint8_t* hbt_ok, const double* hbt_x,
              const double* hbt_y, double hbt_pitch, double hbt_cost, double* out, int32_t* n_bad,
              double* scratch, void* stream) {
  if (n_net < 0 || !net_ptr || !out || !n_bad || !scratch ||
      (n_net > 0 && (!pin_inst || !ox_top || !oy_top || !ox_bot || !oy_bot || !w_top || !h_top ||
                     !w_bot || !h_bot || !die || !rot || !x || !y || !hbt_ok || !hbt_x || !hbt_y))) {
    set_error("score: bad args");
    return P3D_ERR_ARG;
  }
  ScoreArgs a{};
  a.n_net = n_net; a.net_ptr = net_ptr; a.pin_inst = pin_inst;
  a.ox_top = ox_top; a.oy_top = oy_top; a.ox_bot = ox_bot; a.oy_bot = oy_bot;
  a.w_top = w_top; a.h_top = h_top; a.w_bot = w_bot; a.h_bot = h_bot;
  a.die = die; a.rot = rot; a.x = x; a.y = y;
  a.hbt_ok = hbt_ok; a.hbt_x = hbt_x; a.hbt_y = hbt_y;
  a.half = hbt_pitch / 2;
  a.cost = hbt_cost;
  a.counter = reinterpret_cast<unsigned int*>(scratch);
  a.partials = scratch + 8;
  a.n_bad = n_bad;
  a.out = out;
  if (n_net == 0) { cudaMemsetAsync(out, 0, 3 * sizeof(double), STREAM(stream)); return check_launch("score"); }
  launch_score(a, STREAM(stream));
  return check_launch("score");
}

int p3d_gp2d_wirelength_ex(int32_t n_net, int32_t n_pin, int32_t n_obj, const int32_t* net_ptr,
                           const int32_t* pin_obj, const uint8_t* pin_top, const double* pin_ox,
                           const double* pin_oy, const int32_t* pin_slot,
                           const int32_t* obj_slot_ptr, const double* pos,
                           const double* gamma_dev, const int32_t* halt, double* value,
                           double* wl_grad, double* scratch, void* stream) {
  if (n_net < 0 || n_pin < 0 || n_obj < 0 || !net_ptr || !pos || !value || !wl_grad || !scratch ||
      (n_pin > 0 && (!pin_obj || !pin_top || !pin_ox || !pin_oy || !pin_slot)) || !obj_slot_ptr ||
      !gamma_dev) {
    set_error("gp2d_wirelength_ex: bad args");
    return P3D_ERR_ARG;
  }
  Gp2dWlArgs a{};
  a.n_net = n_net; a.n_obj = n_obj;
  a.net_ptr = net_ptr; a.pin_obj = pin_obj; a.pin_top = pin_top;
  a.pin_ox = pin_ox; a.pin_oy = pin_oy; a.pin_slot = pin_slot; a.obj_slot_ptr = obj_slot_ptr;
  a.pos = pos; a.gamma = 0.0;
  a.gamma_ptr = gamma_dev; a.halt = halt;
  a.rec = scratch;
  a.counter = reinterpret_cast<unsigned int*>(scratch + 2 * (long long)n_pin);
  a.partials = scratch + 2 * (long long)n_pin + 8;
  a.value = value;
  launch_gp2d_wl(a, wl_grad, STREAM(stream));
  return check_launch("gp2d_wirelength_ex");
}

size_t p3d_sizeof_gp2d_ctl(void) { return sizeof(p3d_gp2d_ctl); }
size_t p3d_sizeof_gp2d_state(void) { return sizeof(p3d_gp2d_state); }

static bool bad_gp2d(const p3d_gp2d_ctl* c) {
  if (!c || c->n_obj < 0 || !c->st || !c->u || !c->v || !c->partials || c->nblk < 1 ||
      c->nblk > kMaxBlocks || (c->n_obj > 0 && (!c->layer || !c->size_w || !c->size_h ||
                                                 !c->charge || !c->is_macro || !c->degree)) ||
      (c->max_iters > 0 && (!c->gamma_tab || !c->log)) || !c->wl_grad || !c->dens_grad ||
      !c->wl_value || !c->ovfl || !c->prev_wl || !c->prev_dens || !c->pre) {
    set_error("invalid p3d_gp2d_ctl descriptor");
    return true;
  }
  return false;
}

int p3d_gp2d_init(const p3d_gp2d_ctl* c, const double* pos0, void* stream) {
  if (bad_gp2d(c) || !pos0) return P3D_ERR_ARG;
  return gp2d_init(*c, pos0, STREAM(stream));
}

int p3d_gp2d_step(const p3d_gp2d_ctl* c, void* stream) {
  if (bad_gp2d(c)) return P3D_ERR_ARG;
  return gp2d_step(*c, STREAM(stream));
}

int p3d_gp2d_project(const p3d_gp2d_ctl* c, const double* in, double* out, void* stream) {
  if (bad_gp2d(c) || !in || !out) return P3D_ERR_ARG;
  return gp2d_project(*c, in, out, STREAM(stream));
}

int p3d_gp2d_layer_xy(int32_t n, const int32_t* idx, const double* pos, int32_t n_obj, double* x,
                      double* y, const int32_t* halt, void* stream) {
  if (n < 0 || n_obj < 0 || (n > 0 && (!idx || !pos || !x || !y))) { set_error("gp2d_layer_xy: bad args"); return P3D_ERR_ARG; }
  if (n == 0) return P3D_OK;
  launch_gp2d_layer_xy(n, idx, pos, n_obj, x, y, halt, STREAM(stream));
  return check_launch("gp2d_layer_xy");
}

int p3d_gp2d_layer_force(int32_t n, const int32_t* idx, const double* force, double* dens_grad,
                         const int32_t* halt, void* stream) {
  if (n < 0 || (n > 0 && (!idx || !force || !dens_grad))) { set_error("gp2d_layer_force: bad args"); return P3D_ERR_ARG; }
  if (n == 0) return P3D_OK;
  launch_gp2d_layer_force(n, idx, force, dens_grad, halt, STREAM(stream));
  return check_launch("gp2d_layer_force");
}

int p3d_dynamic_size(int32_t n, const double* w_top, const double* h_top, const double* w_bot,
                     const double* h_bot, const uint8_t* is_macro, const double* z, double dz,
                     double* w, double* h, void* stream) {
  if (n < 0 || (n > 0 && (!w_top || !h_top || !w_bot || !h_bot || !is_macro || !z || !w || !h))) {
    set_error("dynamic_size: bad args");
    return P3D_ERR_ARG;
  }
  if (n == 0) return P3D_OK;
  launch_dynamic_size(n, w_top, h_top, w_bot, h_bot, is_macro, z, dz, w, h, STREAM(stream));
  return check_launch("dynamic_size");
}

int p3d_prefix_sum_3d(int32_t nx, int32_t ny, int32_t nz, int32_t reverse, double* a,
                      void* stream) {
  if (nx < 1 || ny < 1 || nz < 1 || !a) { set_error("prefix_sum_3d: bad args"); return P3D_ERR_ARG; }
  for (int ax = 0; ax < 3; ++ax) launch_axis_scan(nx, ny, nz, ax, reverse != 0, a, STREAM(stream));
  return check_launch("prefix_sum_3d");
}

int p3d_overflow(int64_t n, const double* rho, double rho_t, double bin_vol,
                 double movable_volume, double* out, double* scratch, void* stream) {
  if (n < 1 || !rho || !out || !scratch) { set_error("overflow: bad args"); return P3D_ERR_ARG; }
  launch_overflow_d(n, rho, rho_t, bin_vol / movable_volume, scratch, out, STREAM(stream));
  return check_launch("overflow");
}

int p3d_net_spans(int32_t n_net, const int64_t* cnt, const double* min1, const double* max1,
                  const double* full_min, const double* full_max, double* top, double* bot,
                  double* full, void* stream) {
  if (n_net < 0 || (n_net > 0 && (!cnt || !min1 || !max1 || !full_min || !full_max || !top || !bot || !full))) {
    set_error("net_spans: bad args");
    return P3D_ERR_ARG;
  }
  if (n_net == 0) return P3D_OK;
  launch_spans(n_net, cnt, min1, max1, full_min, full_max, top, bot, full, STREAM(stream));
  return check_launch("net_spans");
}

int p3d_nesterov_op(int32_t op, int64_t n, const double* v, const double* vp, const double* g,
                    const double* ref, double s, double* out, double* scratch, void* stream) {
  if (n < 1 || !out || !g || (op == 0 && (!v || !vp || !ref || !scratch)) ||
      (op == 1 && !scratch) || (op == 2 && !v) || op < 0 || op > 2) {
    set_error("nesterov_op: bad args");
    return P3D_ERR_ARG;
  }
  if (op == 0) launch_bb_norms(n, v, vp, g, ref, scratch, out, STREAM(stream));
  else if (op == 1) launch_absmax(n, g, scratch, out, STREAM(stream));
  else launch_axpy(n, v, s, g, ref, out, STREAM(stream));
  return check_launch("nesterov_op");
}

int p3d_rebalance(int32_t n, const double* area_top, const double* area_bot,
                  const int32_t* order_top, const int32_t* order_bot, uint8_t* delta,
                  double cap_top, double cap_bot, double* out, void* stream) {
  if (n < 0 || !out || (n > 0 && (!area_top || !area_bot || !order_top || !order_bot || !delta))) {
    set_error("rebalance: bad args");
    return P3D_ERR_ARG;
  }
  RebalanceArgs a{n, area_top, area_bot, order_top, order_bot, delta, cap_top, cap_bot, out};
  launch_rebalance(a, STREAM(stream));
  return check_launch("rebalance");
}

int p3d_check_objects(int32_t n_inst, int32_t n_net, const uint8_t* die, const int32_t* rot,
                      const double* x, const double* y, const uint8_t* is_macro,
                      const double* w_top, const double* h_top, const double* w_bot,
                      const double* h_bot, const int32_t* net_ptr, const int32_t* pin_inst,
                      const uint8_t* hbt_ok, const double* hbt_x, const double* hbt_y,
                      double die_w, double die_h, double row_top, double row_bot, double site_w,
                      double pitch, double tol, uint8_t* inst_flags, uint8_t* net_flags,
                      double* box, double* area, double* scratch, void* stream) {
  if (n_inst < 1 || n_net < 0 || !die || !rot || !x || !y || !is_macro || !w_top || !h_top ||
      !w_bot || !h_bot || !inst_flags || !box || !area || !scratch ||
      (n_net > 0 && (!net_ptr || !pin_inst || !hbt_ok || !hbt_x || !hbt_y || !net_flags)) ||
      !(row_top > 0) || !(row_bot > 0) || !(site_w > 0)) {
    set_error("check_objects: bad args");
    return P3D_ERR_ARG;
  }
  CheckArgs a{};
  a.n_inst = n_inst; a.n_net = n_net; a.die = die; a.rot = rot; a.x = x; a.y = y;
  a.is_macro = is_macro; a.w_top = w_top; a.h_top = h_top; a.w_bot = w_bot; a.h_bot = h_bot;
  a.net_ptr = net_ptr; a.pin_inst = pin_inst; a.hbt_ok = hbt_ok; a.hbt_x = hbt_x; a.hbt_y = hbt_y;
  a.die_w = die_w; a.die_h = die_h; a.row_top = row_top; a.row_bot = row_bot; a.site_w = site_w;
  a.pitch = pitch; a.tol = tol; a.inst_flags = inst_flags; a.net_flags = net_flags; a.box = box;
  a.area = area;
  a.counter = reinterpret_cast<unsigned int*>(scratch);
  a.partials = scratch + 8;
  launch_check(a, STREAM(stream));
  return check_launch("check_objects");
}

int p3d_pair_search(int32_t phase, int32_t n, const double* box, const uint8_t* member,
                    double bucket, int32_t nbx, int32_t nby, int32_t mode, double min_cc,
                    double tol, int32_t* count, int32_t* start, int32_t* cursor, int32_t* list,
                    int32_t* out, int32_t cap, int32_t* n_out, void* stream) {
  if (phase < 0 || phase > 2 || n < 0 || nbx < 1 || nby < 1 || !(bucket > 0) || mode < 0 ||
      mode > 1 || (n > 0 && (!box || !member)) || (phase == 0 && !count) ||
      (phase == 1 && (!cursor || !list)) || (phase == 2 && (!start || !list || !out || !n_out || cap < 0))) {
    set_error("pair_search: bad args");
    return P3D_ERR_ARG;
  }
  PairArgs a{};
  a.n = n; a.box = box; a.member = member; a.bucket = bucket; a.nbx = nbx; a.nby = nby;
  a.mode = mode; a.min_cc = min_cc; a.tol = tol; a.count = count; a.start = start;
  a.cursor = cursor; a.list = list; a.out = out; a.cap_out = cap; a.n_out = n_out;
  if (n == 0) return P3D_OK;
  if (phase == 0) launch_pair_count(a, STREAM(stream));
  else if (phase == 1) launch_pair_fill(a, STREAM(stream));
  else launch_pair_test(a, STREAM(stream));
  return check_launch("pair_search");
}

int p3d_precondition(int32_t n, const double* gr, double lam, const double* q, const double* deg,
                     const uint8_t* macro, double* out, double* div, void* stream) {
  if (n < 0 || !gr || !q || !deg || !out) { set_error("precondition: bad args"); return P3D_ERR_ARG; }
  if (n == 0) return P3D_OK;
  launch_precondition(n, gr, lam, q, deg, macro, out, div, STREAM(stream));
  return check_launch("precondition");
}

static bool bad_gp(const p3d_gp* gp) {
  // every per-launch grid writes one partial per block into a kMaxBlocks-wide
  // slot: the density kernel runs n_macro + nblk_dens blocks
  if (!gp || !gp->st || !gp->u || !gp->v || !gp->partials || gp->n_obj <= 0 ||
      gp->n_inst < 0 || gp->nblk_obj <= 0 || gp->nblk_obj > kMaxBlocks || gp->nblk_net <= 0 ||
      gp->nblk_net > kMaxBlocks || gp->nblk_dens < 1 || gp->n_macro < 0 ||
      gp->n_macro + gp->nblk_dens > kMaxBlocks) {
    set_error("invalid p3d_gp descriptor");
    return true;
  }
  return bad_grid(&gp->grid);
}

int p3d_gp_init(const p3d_gp* gp, const double* pos0, void* stream) {
  if (bad_gp(gp) || !pos0) return P3D_ERR_ARG;
  return gp_init(*gp, pos0, STREAM(stream));
}

int p3d_gp_iterate(const p3d_gp* gp, void* stream) {
  if (bad_gp(gp)) return P3D_ERR_ARG;
  return gp_iterate(*gp, STREAM(stream));
}

int p3d_gp_iterate_steady(const p3d_gp* gp, void* stream) {
  if (bad_gp(gp)) return P3D_ERR_ARG;
  return gp_iterate(*gp, STREAM(stream), /*steady=*/true);
}

int p3d_gp_iterate_profiled(const p3d_gp* gp, void* stream, float* stage_ms) {
  if (bad_gp(gp) || !stage_ms) return P3D_ERR_ARG;
  return gp_iterate_profiled(*gp, STREAM(stream), stage_ms);
}

int p3d_gp_iterate_marked_overlap(const p3d_gp* gp, void* stream) {
  if (bad_gp(gp)) return P3D_ERR_ARG;
  if (!gp->overlap) { set_error("gp_iterate_marked_overlap: descriptor without overlap"); return P3D_ERR_ARG; }
  return gp_iterate_marked_overlap(*gp, STREAM(stream));
}

int p3d_gp_overlap_times(float* t) {
  if (!t) return P3D_ERR_ARG;
  return gp_overlap_times(t);
}

int p3d_gp_iterate_marked(const p3d_gp* gp, void* stream) {
  if (bad_gp(gp)) return P3D_ERR_ARG;
  return gp_iterate_marked(*gp, STREAM(stream));
}

int p3d_gp_stage_times(float* stage_ms) {
  if (!stage_ms) return P3D_ERR_ARG;
  return gp_stage_times(stage_ms);
}

int p3d_gp_kernels_per_iteration(const p3d_gp* gp) {
  if (bad_gp(gp)) return -1;
  return gp_kernels_per_iteration(*gp);
}

int p3d_gp_evaluate(const p3d_gp* gp, double lam, double gamma, void* stream) {
  if (bad_gp(gp)) return P3D_ERR_ARG;
  return gp_evaluate(*gp, lam, gamma, STREAM(stream));
}

int p3d_gp_density_fx(const p3d_gp* gp, int64_t* out, void* stream) {
  if (bad_gp(gp)) return P3D_ERR_ARG;
  if (!out) { set_error("gp_density_fx: null argument"); return P3D_ERR_ARG; }
  return gp_density_fx(*gp, out, STREAM(stream));
}

int p3d_gp_shard_stage(const p3d_gp* gp, int stage, void* stream) {
  if (!gp || stage < 0 || stage >= P3D_SH_N_STAGES) { set_error("gp_shard_stage: bad stage"); return P3D_ERR_ARG; }
  if (gp->shard_size < 1 || !gp->shard_tot) { set_error("gp_shard_stage: not a sharded problem (shard_size < 1 or no shard_tot)"); return P3D_ERR_ARG; }
  return gp_shard_stage(*gp, stage, STREAM(stream));
}

int p3d_gp_project(const p3d_gp* gp, const double* in, double* out, void* stream) {
  if (bad_gp(gp) || !in || !out) return P3D_ERR_ARG;
  return gp_project(*gp, in, out, STREAM(stream));
}

}  // extern "C"
