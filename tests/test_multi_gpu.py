"""CPU, world_size 2 over gloo: the multi-GPU host logic (element partition,
slice addressing, verification gather, max-over-ranks timing) exercised with
the oracle standing in for the per-device kernel.  The per-slice kernel itself
is covered by tests/test_gpu_parity.py; here the question is only whether the
partition + gather reproduce the unpartitioned result bit-exactly."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, cases, q):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch
    import torch.distributed as dist

    import oracle as O
    import paper_2107_14027_b200 as hf
    from paper_2107_14027_b200 import PhysParams, Precision, StateField
    from paper_2107_14027_b200.multi_gpu import make_slice, partitioned_divergence

    dist.init_process_group("gloo", rank=rank, world_size=world)
    par = PhysParams(1.0 / 1600.0, 2.5, 1.0)
    ok = []
    for (d, p, n, g, fp32, src) in cases:
        U = StateField(d, p, n, g, Precision.fp32 if fp32 else Precision.fp64,
                       O.random_field(d, p, n, g, fp32, 7 + n))

        def cpu_compute(sp, u):  # oracle stand-in for the device kernel on one slice
            return O.oracle_divergence(d, p, sp.n_elem, g, np.ascontiguousarray(u), par.nu, par.zeta, par.T,
                                       (1.0, 1.0, 1.0), src)

        out = partitioned_divergence(U, par, with_source=src, compute=cpu_compute, dist=dist)
        sl = make_slice(hf.problem_for(U, par), world, rank)
        # max-over-ranks reduction used by bench.py for the device time
        t = torch.tensor([float(rank + 1)], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        if rank == 0:
            ref = O.oracle_divergence(d, p, n, g, U.data, par.nu, par.zeta, par.T, (1.0, 1.0, 1.0), src)
            ok.append(bool(np.array_equal(out.data, ref)) and t.item() == world and sl.e_begin == 0)
        else:
            ok.append(sl.e_begin % g == 0 and sl.e_begin > 0)
    dist.barrier()
    dist.destroy_process_group()
    q.put((rank, ok))


@pytest.mark.parametrize("world", [2])
def test_partitioned_equals_unpartitioned_gloo(world):
    cases = [(3, 2, 37, 4, False, True), (3, 3, 16, 8, True, False), (2, 4, 21, 2, False, False)]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, cases, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = dict(q.get(timeout=240) for _ in range(world))
    for pr in procs:
        pr.join(timeout=60)
    assert all(all(v) for v in res.values()), res


def test_slices_tile_the_field():
    import paper_2107_14027_b200 as hf
    from paper_2107_14027_b200 import PhysParams, Precision
    from paper_2107_14027_b200.multi_gpu import all_slices
    for (n, g, world) in [(2343750, 8, 8), (694445, 2, 8), (1000, 16, 4), (5, 4, 8)]:
        pr = hf.make_problem(3, 3, n, g, Precision.fp64, PhysParams())
        sls = all_slices(pr, world)
        assert sls[0].word_offset == 0
        for a, b in zip(sls, sls[1:]):
            assert a.word_end == b.word_offset or b.n_elem == 0
        assert sum(s.n_elem for s in sls) == n
        assert max(s.word_end for s in sls) == hf.field_words(pr)
        sizes = [s.n_elem for s in sls if s.n_elem]
        assert max(sizes) - min(sizes) <= g  # balanced to within one group


# ---------------------------------------------------------------- FR right-hand side: layer slabs + ghost exchange
def _fr_worker(rank, world, port, cases, q, fused=False):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch
    import torch.distributed as dist

    import oracle as O
    import paper_2107_14027_b200 as hf
    from paper_2107_14027_b200 import PhysParams, Precision
    from paper_2107_14027_b200.multi_gpu import fr_residual_slab, make_fr_slab

    dist.init_process_group("gloo", rank=rank, world_size=world)
    par = PhysParams(1.0 / 1600.0, 2.5, 1.0)
    ok = []
    for (d, p, dims, g, src) in cases:
        n = int(np.prod(dims))
        U = O.random_field(d, p, n, g, False, 31 + n)
        pr = hf.make_problem(d, p, n, g, Precision.fp64, par, with_source=src)
        sl = make_fr_slab(pr, dims, world, rank)
        gw = hf.field_words(pr) // (n // g)
        fw = hf.face_words(pr) // (n // g)
        e0, e1 = sl.e_begin, sl.e_begin + sl.n_elem
        jac = (1.0, 1.0, 1.0)

        class CpuOps:  # oracle stand-ins for the three device kernels (test infrastructure)
            @staticmethod
            def divergence(sp, u, out):
                out[:] = torch.from_numpy(O.oracle_divergence(d, p, sp.n_elem, g, u.numpy(), par.nu, par.zeta, par.T,
                                                              jac, src))

            @staticmethod
            def project(sp, u, uf):
                uf[:] = torch.from_numpy(O.project_faces(d, p, sp.n_elem, g, u.numpy()))

            @staticmethod
            def correct(sp, mesh, uf, out, glo, ghi):
                Ufg = np.zeros(hf.face_words(pr))
                Ufg[e0 // g * fw:e1 // g * fw] = uf.numpy()
                if glo is not None:
                    lo = (e0 - sl.layer) % n
                    hi = e1 % n
                    Ufg[lo // g * fw:(lo + sl.layer) // g * fw] = glo.numpy()
                    Ufg[hi // g * fw:(hi + sl.layer) // g * fw] = ghi.numpy()
                outg = np.zeros(hf.field_words(pr))
                outg[e0 // g * gw:e1 // g * gw] = out.numpy()
                O.fr_correct(d, p, g, dims, Ufg, outg, par.nu, par.zeta, par.T, jac, e0, e1)
                out[:] = torch.from_numpy(outg[e0 // g * gw:e1 // g * gw])

        if fused:  # the device drivers' order: faces with the divergence, then the exchange
            CpuOps.divergence_faces = staticmethod(
                lambda sp, u_, out_, uf_: (CpuOps.divergence(sp, u_, out_), CpuOps.project(sp, u_, uf_)))

        u = torch.from_numpy(U[e0 // g * gw:e1 // g * gw].copy())
        out = torch.zeros_like(u)
        uf = torch.zeros(hf.face_words(sl.problem), dtype=torch.float64)
        glo = torch.zeros(sl.face_layer_words, dtype=torch.float64)
        ghi = torch.zeros(sl.face_layer_words, dtype=torch.float64)
        fr_residual_slab(sl, u, out, uf, glo, ghi, dist=dist, ops=CpuOps)
        parts = [None] * world
        dist.all_gather_object(parts, (e0, e1, out.numpy()))
        if rank == 0:
            full = np.zeros(hf.field_words(pr))
            for a, b, arr in parts:
                full[a // g * gw:b // g * gw] = arr
            ref = O.fr_residual(d, p, dims, g, U, par.nu, par.zeta, par.T, jac, src)
            ok.append(float(np.max(np.abs(full - ref))))
    dist.barrier()
    dist.destroy_process_group()
    q.put((rank, ok))


@pytest.mark.parametrize("world,fused", [(2, False), (3, False), (2, True)])
def test_fr_slabs_with_ghost_exchange_gloo(world, fused):
    cases = [(3, 2, (2, 2, 6), 4, True), (3, 3, (3, 2, 3), 2, False), (2, 4, (4, 6), 4, True)]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_fr_worker, args=(r, world, port, cases, q, fused)) for r in range(world)]
    for pr_ in procs:
        pr_.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for pr_ in procs:
        pr_.join(timeout=60)
    assert len(res[0]) == len(cases) and max(res[0]) == 0.0, res
