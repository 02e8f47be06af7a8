"""Element-partitioned multi-GPU driver.

Elements are independent on this path: the divergence of element e reads only
element e (oracle.hpp:30-58).  A field is therefore split into contiguous,
group-aligned slices (``hf_partition``); each slice is itself a valid field
with the same AoSoA group (layout.hpp:128-133), and every rank / device runs
the fused kernel on its own slice.  There is no collective on the data path.
``torch.distributed`` is used only for plumbing: a barrier, the max-over-ranks
of the device time, and -- for verification only -- gathering slices.

One process per GPU (torchrun) is the deployment model; ``Slice`` and
``gather_field`` are backend-agnostic so the same host logic is exercised with
the ``gloo`` backend on CPU in tests/test_multi_gpu.py.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, Optional

import numpy as np

from . import hexfuse as H


@dataclass
class Slice:
    rank: int
    world: int
    e_begin: int        # first global element of the slice
    n_elem: int         # elements in the slice
    word_offset: int    # first word of the slice inside the global field
    n_words: int        # padded words of the slice (n_groups * group_words)
    problem: object     # hf_problem describing the slice alone

    @property
    def word_end(self) -> int:
        return self.word_offset + self.n_words


def make_slice(pr, world: int, rank: int) -> Slice:
    e0, ne, wo = H.partition(pr, world, rank)
    sp = H.make_problem(pr.d, pr.p, ne, pr.group, pr.precision,
                        H.PhysParams(pr.nu, pr.zeta, pr.T), tuple(pr.jac), bool(pr.with_source), pr.method)
    nw = H.field_words(sp) if ne > 0 else 0
    return Slice(rank, world, e0, ne, wo, nw, sp)


def all_slices(pr, world: int):
    return [make_slice(pr, world, r) for r in range(world)]


def run_slice_on_device(sl: Slice, u_slice, out_slice, stream=None) -> None:
    """The fused kernel on one slice (device buffers of sl.n_words words)."""
    if sl.n_elem > 0:
        H.fused_divergence_device(sl.problem, u_slice, out_slice, stream)


def gather_field(pr, local_out: np.ndarray, sl: Slice, dist=None) -> Optional[np.ndarray]:
    """Verification-only host gather of every rank's slice result into the full
    field on rank 0 (padding of the global field stays zero).  Uses
    all_gather_object so it works on gloo (CPU) and nccl alike."""
    if dist is None:
        import torch.distributed as dist
    parts = [None] * sl.world
    dist.all_gather_object(parts, (sl.word_offset, np.asarray(local_out[: sl.n_words])))
    if sl.rank != 0:
        return None
    full = np.zeros(H.field_words(pr))
    for off, arr in parts:
        # slice padding (only in the globally-last slice) is the global padding
        full[off: off + arr.size] = arr
    return full


def partitioned_divergence(U: "H.StateField", params: "H.PhysParams", jac=(1.0, 1.0, 1.0), with_source=False,
                           compute: Optional[Callable] = None, dist=None):
    """Each rank computes its slice of ``fused_divergence(U, ...)``; rank 0 gets
    the assembled StateField (others get None).  ``compute(slice_problem,
    u_words) -> out_words`` defaults to the B200 host-buffer path; tests pass a
    CPU stand-in to exercise the partition logic without a GPU."""
    if dist is None:
        import torch.distributed as dist
    world, rank = dist.get_world_size(), dist.get_rank()
    pr = H.problem_for(U, params, jac, with_source)
    sl = make_slice(pr, world, rank)
    u_local = U.data[sl.word_offset: sl.word_end]
    if compute is None:
        def compute(sp, u):
            src = H.StateField(U.d, U.p, sl.n_elem, U.group, U.precision, u)
            return H.fused_divergence(src, params, jac, with_source).data
    out_local = compute(sl.problem, u_local) if sl.n_elem > 0 else np.zeros(0)
    full = gather_field(pr, out_local, sl, dist)
    if full is None:
        return None
    return H.StateField(U.d, U.p, U.n_elem, U.group, U.precision, full)


# ------------------------------------------------------------------------------------------------
# The FR right-hand side on a layer-partitioned periodic mesh: the
# first place the path has a real exchange step.  Stage 4 (the common interface
# flux) reads the neighbouring element's face values, so a rank that owns a slab
# of whole element layers needs the faces of the layer just below and just above
# it -- the ghost layers.  They travel as point-to-point NCCL messages (NVLink /
# NVSwitch on one node; gloo on CPU in the tests), overlapped with the fused
# divergence kernel, which needs no halo.
# ------------------------------------------------------------------------------------------------
@dataclass
class FrSlab:
    rank: int
    world: int
    d: int
    dims: tuple
    layer: int           # elements per layer
    l_begin: int         # first layer of the slab
    l_end: int
    e_begin: int
    n_elem: int
    problem: object      # hf_problem of the slab (the global problem's d, p, group, params)
    face_layer_words: int  # face words of one layer

    @property
    def n_layers(self) -> int:
        return self.l_end - self.l_begin


def make_fr_slab(pr, dims, world: int, rank: int) -> FrSlab:
    """Rank `rank`'s contiguous run of whole element layers (the last mesh axis).
    Layers must be whole AoSoA groups (layer % group == 0) and every rank needs at
    least one layer."""
    d = pr.d
    dims = tuple(int(x) for x in dims[:d])
    layer = dims[0] * dims[1] if d == 3 else dims[0]
    n_layers = dims[-1]
    if layer % pr.group:
        raise H.HexfuseInvalid("FrSlab: an element layer must be a whole number of AoSoA groups")
    if world > n_layers:
        raise H.HexfuseInvalid("FrSlab: more ranks than element layers")
    l0 = (n_layers * rank) // world
    l1 = (n_layers * (rank + 1)) // world
    sp = H.make_problem(d, pr.p, (l1 - l0) * layer, pr.group, pr.precision,
                        H.PhysParams(pr.nu, pr.zeta, pr.T), tuple(pr.jac), bool(pr.with_source))
    one = H.make_problem(d, pr.p, layer, pr.group, pr.precision, H.PhysParams(pr.nu, pr.zeta, pr.T))
    return FrSlab(rank, world, d, dims, layer, l0, l1, l0 * layer, (l1 - l0) * layer, sp, H.face_words(one))


def exchange_ghost_layers(sl: FrSlab, uf, ghost_lo, ghost_hi, dist=None):
    """Send this slab's first face layer to rank-1 (its ghost_hi) and its last to
    rank+1 (its ghost_lo); receive ours.  Periodic ring; non-blocking (returns the
    request list).  uf / ghost_* are 1-D tensors (CUDA for NCCL, CPU for gloo)."""
    if dist is None:
        import torch.distributed as dist
    w = sl.face_layer_words
    lo_rank, hi_rank = (sl.rank - 1) % sl.world, (sl.rank + 1) % sl.world
    first = uf[:w].contiguous()
    last = uf[(sl.n_layers - 1) * w: sl.n_layers * w].contiguous()
    # Message order = matching order per peer (NCCL has no tags): with two ranks both
    # neighbours are the same peer, whose first layer is our ghost_hi and last our ghost_lo,
    # so every rank posts "first layer -> ghost_hi" before "last layer -> ghost_lo".
    ops = [dist.P2POp(dist.isend, first, lo_rank, tag=0), dist.P2POp(dist.isend, last, hi_rank, tag=1),
           dist.P2POp(dist.irecv, ghost_hi, hi_rank, tag=0), dist.P2POp(dist.irecv, ghost_lo, lo_rank, tag=1)]
    return dist.batch_isend_irecv(ops)


class FrOps:
    """The per-rank kernels of the FR right-hand side: the B200 library by default.
    Tests substitute CPU stand-ins (oracle) to exercise the partition and halo logic."""

    @staticmethod
    def divergence(sp, u, out):
        H.fused_divergence_device(sp, u, out)

    @staticmethod
    def project(sp, u, uf):
        H.fr_project_device(sp, u, uf)

    @staticmethod
    def divergence_faces(sp, u, out, uf):
        H.fr_divergence_faces_device(sp, u, uf, out)

    @staticmethod
    def correct(sp, mesh, uf, out, ghost_lo, ghost_hi):
        H.fr_correct_device(sp, mesh, uf, out, ghost_lo, ghost_hi)


def fr_residual_slab(sl: FrSlab, u, out, uf, ghost_lo, ghost_hi, dist=None, ops=FrOps):
    """Stages 1-6 on one rank's slab, then the ghost-layer exchange and the
    interface corrections.  With ``ops.divergence_faces`` (the device default:
    faces written by the fused kernel, one pass over U) the exchange follows
    that kernel; otherwise the faces are projected first and the exchange runs
    while the fused divergence computes.  With world == 1 the mesh wraps onto
    itself and no message is sent."""
    fused = getattr(ops, "divergence_faces", None)
    if fused is not None:
        fused(sl.problem, u, out, uf)
    else:
        ops.project(sl.problem, u, uf)
    reqs = []
    if sl.world > 1:
        if hasattr(u, "is_cuda") and u.is_cuda:
            import torch
            torch.cuda.current_stream().synchronize()  # faces complete before NCCL reads them
        reqs = exchange_ghost_layers(sl, uf, ghost_lo, ghost_hi, dist)
    if fused is None:
        ops.divergence(sl.problem, u, out)
    for r in reqs:
        r.wait()
    mesh = H.make_mesh(sl.dims, sl.d, sl.e_begin, sl.n_elem, sl.layer if sl.world > 1 else 0)
    ops.correct(sl.problem, mesh, uf, out, ghost_lo if sl.world > 1 else None, ghost_hi if sl.world > 1 else None)


class FrPeers:
    """The neighbouring ranks' face arrays mapped into this process (CUDA IPC:
    peer memory over NVLink / NVSwitch).  With them, hf_fr_correct reads the
    ghost layers straight from the neighbours' memory -- the exchange and the
    interface kernel are one kernel, with no copy and no NCCL call on the data
    path; ``torch.distributed`` only orders the steps (barriers)."""

    def __init__(self, sl: FrSlab, uf, dist=None):
        if dist is None:
            import torch.distributed as dist
        self.sl = sl
        self._opened = []
        handle, off = H.ipc_handle(uf)
        table = [None] * sl.world
        dist.all_gather_object(table, (handle, off, sl.n_layers))
        wb = uf.element_size()
        lo, hi = (sl.rank - 1) % sl.world, (sl.rank + 1) % sl.world
        base = {}
        for r in {lo, hi}:
            h, o, _ = table[r]
            if r == sl.rank:  # world == 1: our own array
                base[r] = int(uf.data_ptr())
            else:
                ptr = H.ipc_open(h)
                self._opened.append(ptr)
                base[r] = ptr + o
        w = sl.face_layer_words
        self.ghost_lo = base[lo] + (table[lo][2] - 1) * w * wb  # last layer below us
        self.ghost_hi = base[hi]                                 # first layer above us

    def close(self):
        for ptr in self._opened:
            H.ipc_close(ptr)
        self._opened = []


def fr_residual_slab_peer(sl: FrSlab, u, out, uf, peers: FrPeers, dist=None):
    """Stages 1-6 on one rank's slab with the ghost layers read from peer memory.
    Barriers: every rank's faces are projected before anyone corrects, and every
    correction has finished before anyone projects the next step's faces."""
    if dist is None:
        import torch.distributed as dist
    import torch
    H.fr_divergence_faces_device(sl.problem, u, uf, out)  # stages 1+2+3+6, one pass over U
    torch.cuda.current_stream().synchronize()
    dist.barrier()
    mesh = H.make_mesh(sl.dims, sl.d, sl.e_begin, sl.n_elem, sl.layer)
    H.fr_correct_device(sl.problem, mesh, uf, out, peers.ghost_lo, peers.ghost_hi)
    torch.cuda.current_stream().synchronize()
    dist.barrier()
