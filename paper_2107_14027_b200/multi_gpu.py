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
