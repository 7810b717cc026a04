"""Sharded GP loop (north_star's config-4 path): one placement
partitioned over the ranks of a torch.distributed group, one GPU per rank.

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
    ADVANCE           Nesterov step on own objects
    [all-reduce]      |v_new - v|^2;   [all-gather] own pos4 slabs for K1

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
from .gp import Gp3dProblem

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

    def all_reduce(self, t, op=None):
        if not self.on:
            return
        op = dist.ReduceOp.SUM if op is None else op
        if self.nccl:
            dist.all_reduce(t, op=op)
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
                 comm=None):
        self.comm = comm or ShardComm()
        self.prob = Gp3dProblem(design, grid, fillers, cfg, rot, max_iters=max_iters,
                                precision=precision, shard=(self.comm.rank, self.comm.world))
        p = self.prob
        off = _lib.LoopState.dv2_next.offset
        self._dv2 = p.t_st[off: off + 8].view(torch.float64)
        self._tot16 = p.t_shard_tot[:16]
        self._tot_max = p.t_shard_tot[16:17]
        self._norms = p.t_shard_tot[20:23]

    def _stage(self, name):
        _lib.call("p3d_gp_shard_stage", _lib.byref(self.prob.gp), STAGE[name], _lib.stream_ptr())

    def init_loop(self, pos0):
        self.prob.init_loop(pos0)

    def iterate(self, n=1, marks=None):
        """n sharded iterations; `marks` (a list) collects (label, cuda Event)
        after every stage / collective for attribution (eager runs only)."""
        p, c = self.prob, self.comm

        def mark(label):
            if marks is not None:
                e = torch.cuda.Event(enable_timing=True)
                e.record()
                marks.append((label, e))

        for _ in range(n):
            mark("start")
            self._stage("NET")
            self._stage("GATHER")
            mark("K1")
            c.reduce_scatter_chunks(p.t_inst_g, 4 * p.inst_slab)  # own instance slab
            mark("comm")
            self._stage("NORMS")
            c.all_reduce(self._norms)
            self._stage("NORMS_FINAL")
            mark("comm")
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
            self._stage("STEP0")
            c.all_reduce(self._tot_max, dist.ReduceOp.MAX if c.on else None)
            self._stage("STEP0_CONTROL")
            mark("comm")
            self._stage("ADVANCE")
            mark("K5")
            c.all_reduce(self._dv2)
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

    def capture(self, iters_per_graph=1):
        """CUDA graph of `iters_per_graph` sharded iterations, collectives
        included (nccl only: gloo stages through host memory).  Replaying it
        removes the per-stage host launch cost."""
        if self.comm.on and not self.comm.nccl:
            raise RuntimeError("graph capture needs the nccl backend")
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s), torch.cuda.graph(g, stream=s):
            self.iterate(iters_per_graph)
        torch.cuda.current_stream().wait_stream(s)
        return g

    def run(self, pos0, poll_every=8, use_graph=False):
        """Initialise and run to completion (max_iters or an exit)."""
        self.init_loop(pos0)
        step = self.iterate
        if use_graph:
            graph = self.capture(1)
            step = lambda n: [graph.replay() for _ in range(n)]  # noqa: E731
        done = 0
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
        return full.reshape(3, O).t().contiguous()

    def log_rows(self, n):
        return self.prob.log_rows(n)
