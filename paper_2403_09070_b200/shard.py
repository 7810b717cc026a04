"""Sharded GP loop (north_star's config-4 path): one placement
partitioned over the ranks of a torch.distributed group, one GPU per rank.

Default (halo mode, partition.py): instances are renumbered so connected
instances are contiguous (label propagation over the netlist), each rank owns
an instance slab and evaluates every net touching it (a net spanning several
ranks runs on each, each keeping its own pins' gradients; its value is counted
once, by its first pin's owner), so the per-instance WL sums are complete on
their owner and only three exchanges remain per iteration:

    [all-to-all]   positions of the halo: each rank receives the pos4 rows of the
                   remote instances of its nets (static lists) -- instead of every
                   position on every rank; at the start of the iteration, next
                   to the density branch (which needs only the rank's own rows)
    [all-reduce]   the three L1 norms (Eq. 17)
    [all-reduce]   rho, int64 fixed point (exact: the single-GPU map bit for bit),
                   on its own communicator (the density branch's side stream)
    [all-reduce]   the density totals with the last step's |v_new - v|^2,
                   (iteration 0) max |g|

The round-robin mode (halo=False) below deals the K1 warp tasks round-robin
and exchanges full per-instance arrays:

Each rank owns a slab of instances (equal padded size), a slab of fillers and
the K1 warp tasks w with w % world == rank.  Per iteration (gp.py:386-444):

    NET, GATHER       K1 on own nets -> records of own pins; owner partial sums
    [reduce-scatter]  per-instance WL sums inst_g [I][4] (fp64): own slab only
    NORMS             L1 norms over the own slab
    [all-reduce]      the three norms;  NORMS_FINAL: Eq. 17 scale
    SCATTER           K2 on own objects -> partial int64 fixed-point rho
    [all-reduce]      rho (int64: exact, the single-GPU map bit for bit)
    SPECTRAL          K3, replicated (maps are small and L2-resident)
    DENS              K4 on own objects -> local totals
    [all-reduce]      totals (energy, L1 norms, |dg|^2, net totals)
    CONTROL           objective, lambda init, log row, best/stop/divergence, BB step
    STEP0 [max] STEP0_CONTROL   iteration 0 only: initial step from max |g|
    ADVANCE           Nesterov step on own objects (|v_new - v|^2 rides along the
                      next all-reduce of totals)
    [all-gather]      own pos4 slabs for K1

All control state is replicated and updated identically on every rank, so the
ranks agree on every branch (stop, divergence, underflow) without host syncs.
ρ-derived quantities equal the single-GPU ones exactly; gradients differ only
by the order of the fp64 owner sums across ranks.

With the nccl backend the collectives run on the device buffers; with gloo
(CPU tests, or several ranks sharing one GPU) they are staged through host
memory.
"""

from __future__ import annotations

import ctypes as C

import numpy as np
import torch
import torch.distributed as dist

from . import _lib
from .dist import object_slabs
from .gp import Gp3dProblem
from .model import ArrayDesign, NetlistArrays
from .partition import HaloPlan, cached_locality_order

STAGE = {name: k for k, name in enumerate(_lib.SH_STAGES)}


class ShardComm:
    """The four collectives the sharded loop needs, on CUDA tensors."""

    def __init__(self, force=False):
        """force: issue the collectives even for a world of one (tests the
        NCCL calls and their graph capture on a single GPU)."""
        self.on = dist.is_initialized() and (dist.get_world_size() > 1 or force)
        self.rank = dist.get_rank() if self.on else 0
        self.world = dist.get_world_size() if self.on else 1
        self.nccl = self.on and dist.get_backend() == "nccl"
        # a second NCCL communicator for the density branch's rho all-reduce:
        # collectives on one communicator run in issue order, so with a single
        # one the WL branch's norm all-reduce would wait for the scatter
        self.side_group = dist.new_group(list(range(self.world))) if self.nccl else None
        if self.nccl:  # initialise both communicators now, not inside a graph capture
            t = torch.zeros(1, device="cuda")
            dist.all_reduce(t)
            dist.all_reduce(t, group=self.side_group)
            torch.cuda.synchronize()

    def all_reduce(self, t, op=None, side=False):
        if not self.on:
            return
        op = dist.ReduceOp.SUM if op is None else op
        if self.nccl:
            dist.all_reduce(t, op=op, group=self.side_group if side else None)
        else:
            h = t.cpu()
            dist.all_reduce(h, op=op)
            t.copy_(h)

    def reduce_scatter_chunks(self, buf, n):
        """buf[r*n:(r+1)*n] <- sum over ranks of that chunk (every rank's own
        chunk; the other chunks are left undefined)."""
        if not self.on or n == 0:
            return
        full = buf[: self.world * n]
        mine = full[self.rank * n:(self.rank + 1) * n]
        if self.nccl:
            dist.reduce_scatter_tensor(mine, full)
        else:
            h = full.cpu()
            dist.all_reduce(h)
            mine.copy_(h[self.rank * n:(self.rank + 1) * n])

    def all_to_all_rows(self, out, inp, out_splits, in_splits):
        """out (rows grouped by source rank) <- rows of inp grouped by
        destination rank (uneven splits)."""
        if not self.on:
            out.copy_(inp)
            return
        if self.nccl:
            dist.all_to_all_single(out, inp, out_splits, in_splits)
        else:
            h = torch.empty(out.shape, dtype=out.dtype)
            dist.all_to_all_single(h, inp.cpu(), out_splits, in_splits)
            out.copy_(h)

    def all_gather_chunks(self, buf, n):
        """buf[:world*n] <- concatenation of every rank's chunk buf[r*n:(r+1)*n]."""
        if not self.on or n == 0:
            return
        full = buf[: self.world * n]
        mine = full[self.rank * n:(self.rank + 1) * n]
        if self.nccl:
            dist.all_gather_into_tensor(full, mine)
        else:
            outs = [torch.empty(n, dtype=buf.dtype) for _ in range(self.world)]
            dist.all_gather(outs, mine.cpu())
            full.copy_(torch.cat(outs))


class ShardedGp3d:
    """run_gp3d's device loop partitioned over the process group."""

    def __init__(self, design, grid, fillers, cfg, rot, max_iters=None, precision=None,
                 comm=None, halo=True):
        self.comm = comm or ShardComm()
        self.halo = bool(halo)
        R, r = self.comm.world, self.comm.rank
        arr = design.arrays()
        I = design.n_insts
        self.perm = self.inv = None
        if self.halo:
            # locality numbering (every rank computes the same, deterministic one)
            perm = cached_locality_order(arr.net_ptr, arr.pin_inst, I)
            inv = np.empty_like(perm)
            inv[perm] = np.arange(I)
            self.perm, self.inv = perm, inv
            pa = NetlistArrays(is_macro=arr.is_macro[perm], w_top=arr.w_top[perm],
                               h_top=arr.h_top[perm], w_bot=arr.w_bot[perm],
                               h_bot=arr.h_bot[perm], net_ptr=arr.net_ptr,
                               pin_inst=inv[arr.pin_inst], ox_top=arr.ox_top,
                               oy_top=arr.oy_top, ox_bot=arr.ox_bot, oy_bot=arr.oy_bot)
            design = ArrayDesign(design.die, design.hbt, pa)
            rot = np.asarray(rot)[perm]
            slab, _, _ = object_slabs(I, fillers.count, r, R)
            self.plan = HaloPlan(pa.net_ptr, pa.pin_inst, I, R, slab)
            shard = (r, R, self.plan)
        else:
            self.plan = None
            shard = (r, R)
        self.prob = Gp3dProblem(design, grid, fillers, cfg, rot, max_iters=max_iters,
                                precision=precision, shard=shard)
        p = self.prob
        self._tot16 = p.t_shard_tot[:16]
        self._tot_max = p.t_shard_tot[16:17]
        self._norms = p.t_shard_tot[20:23]
        if self.halo:
            pl = self.plan
            self._in_splits, self._out_splits = pl.split_sizes(r)
            cat = lambda xs: np.concatenate(xs) if len(xs) else np.zeros(0, np.int64)  # noqa: E731
            self._send_idx = torch.from_numpy(cat(pl.send[r]).astype(np.int64)).cuda()
            self._recv_idx = torch.from_numpy(cat([pl.send[q][r] for q in range(R)])
                                              .astype(np.int64)).cuda()
            self._pos4 = p.t_pos4.view(-1, 4)
            self._send = torch.empty((len(self._send_idx), 4), dtype=torch.float64, device="cuda")
            self._recv = torch.empty((len(self._recv_idx), 4), dtype=torch.float64, device="cuda")

    def exchange_bytes(self):
        """Bytes this rank receives per iteration through its collectives
        (data-path exchanges: owner sums, rho, positions; scalars excluded)."""
        p = self.prob
        rho = 8 * p.grid.n_bins
        if self.halo:
            return {"positions_halo": int(len(self._recv_idx) * 32), "rho_allreduce": rho}
        slab = 32 * p.inst_slab
        return {"owner_sums_reduce_scatter": slab * self.comm.world,
                "positions_allgather": slab * self.comm.world, "rho_allreduce": rho}

    def _halo_exchange(self):
        """pos4 rows of this rank's halo from their owners (all-to-all)."""
        if not self.comm.on:
            return
        torch.index_select(self._pos4, 0, self._send_idx, out=self._send)
        self.comm.all_to_all_rows(self._recv, self._send, self._out_splits, self._in_splits)
        self._pos4.index_copy_(0, self._recv_idx, self._recv)

    def _stage(self, name):
        with torch.cuda.nvtx.range(f"p3d.shard.{name}"):  # free when no profiler listens
            _lib.call("p3d_gp_shard_stage", _lib.byref(self.prob.gp), STAGE[name],
                      _lib.stream_ptr())

    def init_loop(self, pos0):
        # every rank starts from the same positions, so pos4 starts complete
        self.prob.init_loop(self._to_local(pos0))

    def _to_local(self, pos):
        """[O,3] positions in the caller's instance order -> the loop's order."""
        if self.perm is None:
            return pos
        I = self.prob.n_inst
        if isinstance(pos, torch.Tensor):
            idx = torch.from_numpy(self.perm).to(pos.device)
            return torch.cat([pos[:I][idx], pos[I:]])
        pos = np.asarray(pos)
        return np.concatenate([pos[:I][self.perm], pos[I:]])

    def iterate(self, n=1, marks=None, steady=False):
        """n sharded iterations; `marks` (a list) collects (label, cuda Event)
        after every stage / collective for attribution (eager runs only).
        steady=True leaves out the iteration-0 initial step (STEP0, its max
        all-reduce, STEP0_CONTROL): for every iteration after the first."""
        p, c = self.prob, self.comm

        def mark(label):
            if marks is not None:
                e = torch.cuda.Event(enable_timing=True)
                e.record()
                marks.append((label, e))

        # nccl: the density branch (K2, the rho all-reduce, K3) runs on a side
        # stream next to K1 (they are independent until K4), as in the fused
        # loop; every rank issues the collectives in the same program order
        overlap = (c.nccl or not c.on) and marks is None
        if overlap and not hasattr(self, "_side"):
            self._side = torch.cuda.Stream()
        for _ in range(n):
            mark("start")
            if overlap:
                main = torch.cuda.current_stream()
                self._side.wait_stream(main)
                with torch.cuda.stream(self._side):
                    self._stage("SCATTER")
                    c.all_reduce(p.t_rho_fx, side=True)
                    self._stage("SPECTRAL")
            if self.halo:  # the previous step's halo rows, overlapping the density branch
                self._halo_exchange()
                mark("comm")
            self._stage("NET")
            self._stage("GATHER")
            mark("K1")
            if not self.halo:
                c.reduce_scatter_chunks(p.t_inst_g, 4 * p.inst_slab)  # own instance slab
            mark("comm")
            self._stage("NORMS")
            c.all_reduce(self._norms)
            self._stage("NORMS_FINAL")
            mark("comm")
            if overlap:
                main.wait_stream(self._side)
            else:
                self._stage("SCATTER")
                mark("K2")
                c.all_reduce(p.t_rho_fx)
                mark("comm")
                self._stage("SPECTRAL")
                mark("K3")
            self._stage("DENS")
            mark("K4")
            c.all_reduce(self._tot16)
            self._stage("CONTROL")
            if not steady:
                self._stage("STEP0")
                c.all_reduce(self._tot_max, dist.ReduceOp.MAX if c.on else None)
                self._stage("STEP0_CONTROL")
            mark("comm")
            self._stage("ADVANCE")
            mark("K5")
            # |v - v_prev|^2 rides along the next iteration's density totals
            if not self.halo:
                c.all_gather_chunks(p.t_pos4, 4 * p.inst_slab)
                mark("comm")

    @staticmethod
    def attribute(marks):
        """{label: total ms} from the marks of iterate(marks=...)."""
        torch.cuda.synchronize()
        out = {}
        for (_, a), (lab, b) in zip(marks, marks[1:]):
            if lab == "start":
                continue
            out[lab] = out.get(lab, 0.0) + a.elapsed_time(b)
        return out

    def capture(self, iters_per_graph=1, steady=False):
        """CUDA graph of `iters_per_graph` sharded iterations, collectives
        included (nccl only: gloo stages through host memory).  Replaying it
        removes the per-stage host launch cost."""
        if self.comm.on and not self.comm.nccl:
            raise RuntimeError("graph capture needs the nccl backend")
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s), torch.cuda.graph(g, stream=s):
            self.iterate(iters_per_graph, steady=steady)
        torch.cuda.current_stream().wait_stream(s)
        return g

    def stepper(self, iters_per_graph=8):
        """step(n): n iterations replaying captured graphs -- iteration 0 with
        its initial-step stages, every later one without them, in runs of
        `iters_per_graph` steady iterations per replay (the remainder one by
        one).  reset() rewinds to iteration 0 (after init_loop)."""
        g0, gs = self.capture(1), self.capture(1, steady=True)
        gk = self.capture(iters_per_graph, steady=True) if iters_per_graph > 1 else None
        first = [True]

        def step(n=1):
            if n and first[0]:
                g0.replay()
                first[0] = False
                n -= 1
            if gk is not None:
                for _ in range(n // iters_per_graph):
                    gk.replay()
                n %= iters_per_graph
            for _ in range(n):
                gs.replay()

        step.reset = lambda: first.__setitem__(0, True)
        return step

    def run(self, pos0, poll_every=8, use_graph=False):
        """Initialise and run to completion (max_iters or an exit)."""
        self.init_loop(pos0)
        done = 0
        step = self.iterate
        if use_graph:
            step = self.stepper()
        while done < self.prob.max_iters:
            k = min(poll_every, self.prob.max_iters - done)
            step(k)
            done += k
            if self.prob.state().done:
                break
        return self.prob.state()

    def gather_positions(self, which="u"):
        """[O,3] positions (u, v or best) assembled from every rank's slabs."""
        p = self.prob
        src = {"u": p.t_u, "v": p.t_v, "best": p.t_best}[which]
        O = p.n_obj
        full = torch.zeros(3 * O, dtype=torch.float64, device="cuda")
        for lo, hi in (p.sh_i, p.sh_f):
            for c in range(3):
                full[c * O + lo: c * O + hi] = src[c * O + lo: c * O + hi]
        self.comm.all_reduce(full)  # disjoint slabs: the sum is exact
        out = full.reshape(3, O).t().contiguous()
        if self.perm is not None:  # back to the caller's instance order
            I = p.n_inst
            res = out.clone()
            res[torch.from_numpy(self.perm).to(out.device)] = out[:I]
            res[I:] = out[I:]
            out = res
        return out

    def log_rows(self, n):
        return self.prob.log_rows(n)
