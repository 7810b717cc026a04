"""ctypes binding of libp3d.so (the C-ABI in include/p3d.h).

The library is built in-tree (``build.py``); importing this module on a
machine without it, or without a CUDA device, raises immediately — there is
no CPU fallback anywhere in the package.
"""

from __future__ import annotations

import ctypes as C
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
# P3D_LIB_VARIANT=<v> loads libp3d_<v>.so (an A/B build from build.build(variant=...))
_VARIANT = os.environ.get("P3D_LIB_VARIANT", "")
LIB_PATH = os.path.join(_HERE, f"libp3d_{_VARIANT}.so" if _VARIANT else "libp3d.so")

P = C.c_void_p
I32 = C.c_int32
I64 = C.c_int64
D = C.c_double


class Topology(C.Structure):
    _fields_ = [("n_net", I32), ("n_pin", I32), ("n_obj", I32), ("pad0", I32),
                ("net_ptr", P), ("pin_inst", P), ("net_dup", P), ("net_order", P),
                ("pin_slot", P), ("obj_slot_ptr", P)]


class Grid(C.Structure):
    _fields_ = [("nx", I32), ("ny", I32), ("nz", I32), ("pad0", I32),
                ("dx", D), ("dy", D), ("dz", D), ("wb", D), ("hb", D), ("db", D),
                ("bin_vol", D), ("fx_scale", D),
                ("omega", P * 3), ("twiddle", P * 3), ("phase", P * 3)]


class Cloud(C.Structure):
    _fields_ = [("n", I32), ("n_macro", I32), ("x", P), ("y", P), ("z", P), ("w", P),
                ("h", P), ("dep", P), ("weight", P), ("is_macro", P), ("macro_ids", P)]


class LoopState(C.Structure):
    _fields_ = [("it", I32), ("done", I32), ("diverged", I32), ("lam_set", I32),
                ("step_set", I32), ("stop_now", I32), ("best_flag", I32), ("rise", I32),
                ("nonfinite", I32), ("converged", I32), ("eval_only", I32), ("pad0", I32),
                ("lam", D), ("a", D), ("step", D), ("a_new", D), ("mom", D),
                ("prev_ovfl", D), ("prev_value", D), ("last_mu", D), ("best0", D), ("best1", D),
                ("wl_x", D), ("wl_y", D), ("cut", D), ("exact", D), ("ncross", D),
                ("norm_x", D), ("norm_y", D), ("norm_zb", D), ("gz_scale", D),
                ("energy", D), ("ovfl", D), ("value", D), ("wl_value", D), ("l1_wl", D),
                ("l1_dens", D), ("gamma", D), ("lam_eval", D), ("dv2", D), ("dg2", D),
                ("gmax", D), ("dv2_next", D), ("iterations", I32), ("hbt_count", I32),
                ("final_overflow", D), ("wirelength", D), ("counters", C.c_uint32 * 16)]


class Gp(C.Structure):
    _fields_ = [("n_inst", I32), ("n_fill", I32), ("n_obj", I32), ("n_macro", I32),
                ("max_iters", I32), ("divergence_window", I32), ("nblk_obj", I32),
                ("nblk_net", I32), ("wl_f32", I32), ("nblk_dens", I32), ("topo", Topology),
                ("f_n_tasks", I32), ("f_n_generic", I32), ("f_generic_nets", P), ("f_tasks", P), ("f_task_t0", P),
                ("f_net_base", P), ("f_net_deg", P), ("f_net_stride", P), ("f_net_dup", P),
                ("f_pin_inst", P), ("f_pin_off", P), ("f_pin_slot", P), ("grid", Grid),
                ("pin_off", P), ("w_top", P), ("h_top", P), ("w_bot", P), ("h_bot", P),
                ("is_macro", P), ("degree", P), ("fill_w", P), ("fill_h", P), ("fill_z", P),
                ("macro_ids", P), ("gamma_tab", P),
                ("alpha", D), ("target_density", D), ("movable_volume", D),
                ("stop_overflow", D), ("mu_min", D), ("mu_max", D), ("gamma0", D),
                ("gamma1", D), ("min_step", D), ("step_scale", D), ("rho_t_fx", I64),
                ("u", P), ("v", P), ("v_prev", P), ("best", P), ("wl_grad", P),
                ("dens_grad", P), ("pre", P), ("prev_wl", P), ("prev_dens", P), ("prev_q", P),
                ("pin_out", P), ("pin_out_f", P), ("pin_out_fd", P), ("pos4", P), ("inst_g", P), ("rho_fx", P),
                ("ts_n_tiles", I32), ("ts_tiles_x", I32), ("ts_tiles_y", I32), ("ts_margin", I32),
                ("ts_tile_of", P), ("ts_hist", P), ("ts_start", P), ("ts_cursor", P),
                ("ts_order", P), ("ts_rec", P), ("rho", P), ("spec_scratch", P),
                ("maps", P), ("partials", P), ("st", P), ("log", P), ("ovfl_hist", P),
                ("shard_rank", I32), ("shard_size", I32), ("sh_i0", I32), ("sh_i1", I32),
                ("sh_f0", I32), ("sh_f1", I32), ("shard_tot", P), ("overlap", I32),
                ("shard_halo", I32)]

class Gp2dState(C.Structure):
    _fields_ = [("it", I32), ("done", I32), ("diverged", I32), ("converged", I32),
                ("lam_set", I32), ("step_set", I32), ("iterations", I32), ("pad0", I32),
                ("lam", D * 3), ("prev_ovfl", D * 3), ("step", D), ("a", D), ("a_new", D),
                ("mom", D), ("dv2_next", D), ("gamma", D), ("final_overflow", D), ("gmax", D),
                ("counters", C.c_uint32 * 8)]


class Gp2dCtl(C.Structure):
    _fields_ = [("n_obj", I32), ("max_iters", I32), ("n_hbt", I32), ("nblk", I32),
                ("layer", P), ("size_w", P), ("size_h", P), ("charge", P), ("is_macro", P),
                ("degree", P), ("gamma_tab", P), ("die_w", D), ("die_h", D),
                ("stop_overflow", D), ("mu_min", D), ("mu_max", D), ("step_scale", D),
                ("min_step", D), ("pad1", D), ("u", P), ("v", P), ("wl_grad", P),
                ("dens_grad", P), ("wl_value", P), ("ovfl", P), ("prev_wl", P),
                ("prev_dens", P), ("pre", P), ("partials", P), ("log", P), ("st", P)]


SH_STAGES = ("NET", "GATHER", "NORMS", "SCATTER", "SPECTRAL", "DENS", "CONTROL", "STEP0",
             "STEP0_CONTROL", "ADVANCE", "NORMS_FINAL")


_SIGS = {
    "p3d_abi_version": (I32, []),
    "p3d_last_error": (I32, [C.c_char_p, C.c_size_t]),
    "p3d_sizeof_topology": (C.c_size_t, []),
    "p3d_sizeof_grid": (C.c_size_t, []),
    "p3d_sizeof_cloud": (C.c_size_t, []),
    "p3d_sizeof_gp": (C.c_size_t, []),
    "p3d_sizeof_loop_state": (C.c_size_t, []),
    "p3d_gp_partials_doubles": (C.c_size_t, []),
    "p3d_netboxes": (I32, [P, P, P, P, P, P, P, P, P, P, P, P]),
    "p3d_planar_objective_ex": (I32, [P, P, P, P, D, P, P, P, P, P]),
    "p3d_z_cut_penalty_ex": (I32, [P, P, D, P, P, P, P]),
    "p3d_fd_z_gradient": (I32, [P, P, P, P, D, P, P, P]),
    "p3d_gather_pins": (I32, [P, P, P, P]),
    "p3d_pin_coords": (I32, [P, P, P, P, P, D, P, P, P, P, P]),
    "p3d_normalize_z_gradient": (I32, [I32, P, P, P, P, D, P, P, P]),
    "p3d_accumulate_density": (I32, [P, P, P, P]),
    "p3d_fx_to_density": (I32, [I64, P, P, P]),
    "p3d_overflow_fx": (I32, [P, P, D, D, P, P, P]),
    "p3d_spectral": (I32, [P, P, P, P, P, P]),
    "p3d_spectral_from_coef": (I32, [P, P, P, P, P]),
    "p3d_spectral_fx": (I32, [P, P, P, P, D, D, P, P, I32, P]),
    "p3d_density_gather": (I32, [P, P, P, P, P, P, P, P]),
    "p3d_precondition": (I32, [I32, P, D, P, P, P, P, P, P]),
    "p3d_gp_init": (I32, [P, P, P]),
    "p3d_gp_iterate": (I32, [P, P]),
    "p3d_gp_iterate_steady": (I32, [P, P]),
    "p3d_gp_evaluate": (I32, [P, D, D, P]),
    "p3d_gp_project": (I32, [P, P, P, P]),
    "p3d_gp_density_fx": (I32, [P, P, P]),
    "p3d_score": (I32, [I32] + [P] * 17 + [D, D, P, P, P, P]),
    "p3d_gp2d_wirelength": (I32, [I32, I32, I32] + [P] * 8 + [D] + [P] * 4),
    "p3d_gp2d_wirelength_ex": (I32, [I32, I32, I32] + [P] * 14),
    "p3d_sizeof_gp2d_ctl": (C.c_size_t, []),
    "p3d_sizeof_gp2d_state": (C.c_size_t, []),
    "p3d_gp2d_init": (I32, [P, P, P]),
    "p3d_gp2d_step": (I32, [P, P]),
    "p3d_gp2d_project": (I32, [P, P, P, P]),
    "p3d_gp2d_layer_xy": (I32, [I32, P, P, I32, P, P, P, P]),
    "p3d_gp2d_layer_force": (I32, [I32, P, P, P, P, P]),
    "p3d_dynamic_size": (I32, [I32, P, P, P, P, P, P, D, P, P, P]),
    "p3d_prefix_sum_3d": (I32, [I32, I32, I32, I32, P, P]),
    "p3d_overflow": (I32, [I64, P, D, D, D, P, P, P]),
    "p3d_net_spans": (I32, [I32, P, P, P, P, P, P, P, P, P]),
    "p3d_nesterov_op": (I32, [I32, I64, P, P, P, P, D, P, P, P]),
    "p3d_parse_design": (I32, [C.c_char_p, I64, C.POINTER(C.c_void_p)]),
    "p3d_parsed_counts": (I32, [P, P, P]),
    "p3d_parsed_fill": (I32, [P] * 14),
    "p3d_parsed_free": (None, [P]),
    "p3d_rebalance": (I32, [I32, P, P, P, P, P, D, D, P, P]),
    "p3d_check_objects": (I32, [I32, I32] + [P] * 14 + [D] * 7 + [P] * 5),
    "p3d_pair_search": (I32, [I32, I32, P, P, D, I32, I32, I32, D, D, P, P, P, P, P, I32, P, P]),
    "p3d_density_energy_gradient": (I32, [P, P, P, P, P, P, P, P]),
    "p3d_gp_shard_stage": (I32, [P, C.c_int, P]),
    "p3d_gp_iterate_profiled": (I32, [P, P, P]),
    "p3d_gp_kernels_per_iteration": (I32, [P]),
    "p3d_gp_iterate_marked": (I32, [P, P]),
    "p3d_gp_iterate_marked_overlap": (I32, [P, P]),
    "p3d_gp_overlap_times": (I32, [P]),
    "p3d_gp_stage_times": (I32, [P]),
}

EXPORTS = tuple(_SIGS)

_lib = None


def load():
    """Load and type the shared library (raises if it is absent)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"libp3d.so not found at {LIB_PATH}; build it with "
            "`python -c 'import __graft_entry__ as g; g.build()'` (no CPU fallback exists)")
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    for nm, st in (("topology", Topology), ("grid", Grid), ("cloud", Cloud),
                   ("gp", Gp), ("loop_state", LoopState), ("gp2d_ctl", Gp2dCtl),
                   ("gp2d_state", Gp2dState)):
        got = getattr(lib, f"p3d_sizeof_{nm}")()
        if got != C.sizeof(st):
            raise ImportError(f"ABI mismatch: sizeof(p3d_{nm}) C={got} ctypes={C.sizeof(st)}")
    _lib = lib
    return lib


class P3DError(RuntimeError):
    pass


def call(name, *args):
    """Invoke an entry point; non-zero return codes become Python exceptions."""
    lib = load()
    rc = getattr(lib, name)(*args)
    if rc != 0:
        buf = C.create_string_buffer(512)
        lib.p3d_last_error(buf, 512)
        msg = f"{name}: {buf.value.decode(errors='replace')}"
        if rc == 1:
            raise ValueError(msg)
        raise P3DError(msg)


def require_cuda():
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2403_09070_b200 needs a CUDA device (B200); there is no CPU path")


def stream_ptr():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def ptr(t):
    """Device pointer of a tensor (None -> NULL)."""
    if t is None:
        return None
    if not t.is_cuda:
        raise ValueError("expected a CUDA tensor")
    if not t.is_contiguous():
        raise ValueError("expected a contiguous tensor")
    return C.c_void_p(t.data_ptr())


def byref(s):
    return C.byref(s)
