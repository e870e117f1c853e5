"""The sharded path (PAPER.md:138-141 [Sec. 3.2] "data exchange") executed on the GPU.

One B200 per box, so the G > 1 ranks run as an in-process local group (ipr_testing.h): G contexts on one
device, each with its own stream and host thread, exchanging panels by stream-ordered device copies
fenced with events and host barriers -- the engine's column-panel arithmetic, panel-major layouts,
partial gathers, the CRT splits of gathered operands and the tri form's mirror all-to-all, exactly as
over NCCL.  The check is P11: every trace record (rho, delta, decision, certificate) and the returned C
bit-identical to G = 1 for G = 2 and 4 (n = 1024: npad = 1024 for every G, so the tile grid, partial
slots and reduction order do not depend on G).  With two or more GPUs the same comparison runs over
NCCL with one process per GPU (skipped on a one-GPU box)."""
import os
import threading

import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
ipr = pytest.importorskip("paper_1703_02283_b200")

N = 1024
LOW = dict(plateau_ratio=0.7, plateau_arm=0.5, max_iters=40)


def _schedule(name):
    import bench
    return bench.schedule(name, N)


def _solve_world1(A, p, phases, form, cert="fp64"):
    s = ipr.Solver(A, p, phases, 1e-12, form=form, cert=cert)
    s.iterate(300)
    tr, out = s.trace(), s.outcome
    C = s.finalize().cpu().numpy()
    return out, tr, C


def _solve_local(A, p, phases, form, world, grid=None, cert="fp64"):
    grp = ipr.ipr_test_local_group_create(world)
    res = [None] * world
    err = [None] * world

    def rank_main(r):
        try:
            st = torch.cuda.Stream()
            with torch.cuda.stream(st):
                s = ipr.Solver(A, p, phases, 1e-12, stream=st, world=world, rank=r, form=form, local_group=grp,
                               grid=grid, cert=cert)
                s.iterate(300)
                tr, out = s.trace(), s.outcome
                C = torch.empty_like(A)
                s.finalize(C)
                st.synchronize()
                res[r] = (out, tr, C.cpu().numpy())
        except Exception as e:   # noqa: BLE001 -- reported below
            err[r] = e

    th = [threading.Thread(target=rank_main, args=(r,), daemon=True) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(600)
    ipr.ipr_test_local_group_destroy(grp)
    for e in err:
        if e is not None:
            raise e
    return res


def _same_trace(a, b):
    keys = ("phase", "decision", "rho", "delta", "rho_cert", "mant_bits", "digits", "moduli")
    assert len(a) == len(b)
    for x, y in zip(a, b):
        for k in keys:
            vx, vy = x[k], y[k]
            assert (vx == vy) or (vx != vx and vy != vy), (k, x["k"], vx, vy)


CASES = [
    ("literal_fp64", "fp64", 2),
    ("literal_bf16_fp64", "bf16>fp64", 2),
    ("sym_bf16_fp64", "sym:bf16>fp64/cbf16", 2),
    ("sym_fp8_crt", "sym:fp8/cfp8>bf16>fp64crt@a/cbf16", 2),
    ("symtri_headline", "symtri:fp8/cfp8>bf16>fp64crt@a/cbf16", 2),
    ("symtri_bf16_fp64", "symtri:bf16>tf32>fp64/cbf16", 2),
    ("sym_p3_crt", "sym:bf16>fp64crt/cbf16", 3),
    ("symtriz_headline", "symtriz:fp8/cfp8>bf16>fp64crt@a/cbf16", 2),   # R-37: Z_1 mirrored across panels too
]


@pytest.fixture(scope="module")
def A():
    return torch.from_numpy(synth.spd(N, 2.0, 31)).cuda()


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_sharded_bit_identical_to_one_gpu(A, case, world):
    cid, sched, p = case
    form, phases = _schedule(sched)
    out1, tr1, C1 = _solve_world1(A, p, phases, form)
    assert out1 == ipr.IPR_CONVERGED, (cid, out1)
    res = _solve_local(A, p, phases, form, world)
    for r, (out, tr, C) in enumerate(res):
        assert out == out1, (cid, r)
        _same_trace(tr, tr1)
        np.testing.assert_array_equal(C, C1)
    if "crt" in sched:
        assert any(t["moduli"] > 0 for t in tr1)


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("case", [CASES[3], CASES[4], CASES[7]], ids=["sym_fp8_crt", "symtri_headline", "symtriz_headline"])
def test_sharded_crt_certificate_bit_identical_to_one_gpu(A, case, world):
    # IPR_CERT_CRT (R-35) at G > 1: every rank rounds / splits the gathered candidate, computes the
    # column panel Y[:, S_g] exactly (stored K-major: the rows S_g of the symmetric Y), splits those rows,
    # all-gathers the residue planes and the row statistics, and P[:, S_g] with partials in their global
    # slots -- the certified bound, every record and the answer bit-identical to G = 1
    cid, sched, p = case
    form, phases = _schedule(sched)
    out1, tr1, C1 = _solve_world1(A, p, phases, form, cert="crt")
    assert out1 == ipr.IPR_CONVERGED, (cid, out1)
    res = _solve_local(A, p, phases, form, world, cert="crt")
    for r, (out, tr, C) in enumerate(res):
        assert out == out1, (cid, r)
        _same_trace(tr, tr1)
        np.testing.assert_array_equal(C, C1)
    assert tr1[-1]["rho_cert"] <= 1e-12


GRID_CASES = [("literal_fp64", "fp64", 2), ("literal_bf16_fp64", "bf16>fp64", 2), ("literal_tf32_fp64_p3", "tf32>fp64", 3)]


@pytest.mark.parametrize("grid", [(2, 2), (4, 1)], ids=["2x2", "4x1"])
@pytest.mark.parametrize("case", GRID_CASES, ids=[c[0] for c in GRID_CASES])
def test_2d_grid_bit_identical_to_one_gpu(A, case, grid):
    # the true 2-D P_r x P_c option: rank (r, c) owns the block
    # (R_r, S_c) of C and every T_j; Chat row panels gather along grid rows, T_j column panels along grid
    # columns before every GEMM (SUMMA-like), partials from their owners -- the same tiles and K order,
    # so every record and the answer equal G = 1 bit for bit
    cid, sched, p = case
    form, phases = _schedule(sched)
    out1, tr1, C1 = _solve_world1(A, p, phases, form)
    assert out1 == ipr.IPR_CONVERGED
    res = _solve_local(A, p, phases, form, grid[0] * grid[1], grid=grid)
    for out, tr, C in res:
        assert out == out1
        _same_trace(tr, tr1)
        np.testing.assert_array_equal(C, C1)


def test_2d_grid_refuses_other_forms(A):
    form, phases = _schedule("symtri:bf16>fp64/cbf16")
    with pytest.raises(ipr.IprError) as e:
        _solve_local(A, 2, phases, form, 4, grid=(2, 2))
    assert e.value.status == ipr.IPR_E_UNSUPPORTED


def test_local_group_bad_arguments(A):
    with pytest.raises(ipr.IprError):
        ipr.ipr_test_local_group_create(0)
    grp = ipr.ipr_test_local_group_create(2)
    try:
        with pytest.raises(ipr.IprError):
            ipr.Solver(A, 2, [ipr.make_phase("fp64")], world=2, rank=2, local_group=grp)
    finally:
        ipr.ipr_test_local_group_destroy(grp)


def _nccl_rank(rank, world, port, sched, p, q, cert="fp64"):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    obj = [ipr.ipr_nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    A = torch.from_numpy(synth.spd(N, 2.0, 31)).cuda()
    form, phases = _schedule(sched)
    s = ipr.Solver(A, p, phases, 1e-12, world=world, rank=rank, nccl_unique_id=obj[0], form=form, cert=cert)
    s.iterate(300)
    tr = s.trace()
    C = s.finalize().cpu().numpy()
    q.put((rank, s.outcome, tr, C))
    dist.destroy_process_group()


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2, reason="needs >= 2 GPUs (NCCL)")
@pytest.mark.parametrize("case,cert", [(CASES[0], "fp64"), (CASES[4], "fp64"), (CASES[4], "crt")],
                         ids=["literal_fp64", "symtri_headline", "symtri_headline_crt_cert"])
def test_nccl_bit_identical_to_one_gpu(A, case, cert):
    import torch.multiprocessing as mp
    cid, sched, p = case
    form, phases = _schedule(sched)
    out1, tr1, C1 = _solve_world1(A, p, phases, form, cert=cert)
    world = min(torch.cuda.device_count(), 4)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + os.getpid() % 1000
    procs = [ctx.Process(target=_nccl_rank, args=(r, world, port, sched, p, q, cert)) for r in range(world)]
    for pr in procs:
        pr.start()
    got = [q.get(timeout=600) for _ in procs]
    for pr in procs:
        pr.join(60)
    for rank, out, tr, C in got:
        assert out == out1
        _same_trace(tr, tr1)
        np.testing.assert_array_equal(C, C1)


def test_nccl_transport_plumbing_one_gpu():
    # the production transport's calls (dlopen'ed NCCL: init, in-place all-gather, grouped send / recv
    # all-to-all, split) on a 1-rank communicator -- the multi-process test above needs >= 2 GPUs
    ipr.ipr_test_nccl_selftest()


@pytest.mark.parametrize("world", [2])
def test_sharded_host_buffers_crt_certificate(A, world):
    # bench.py's e2e path at N > 1: every rank passes the HOST A (pinned) to ipr_init and a host C to
    # ipr_set_output / ipr_finalize, with the CRT certificate -- the answer bit-identical to the device
    # path at G = 1
    form, phases = _schedule("symtri:fp8/cfp8>bf16>fp64crt@a/cbf16")
    out1, tr1, C1 = _solve_world1(A, 2, phases, form, cert="crt")
    A_host = A.cpu().pin_memory()
    grp = ipr.ipr_test_local_group_create(world)
    res, err = [None] * world, [None] * world

    def rank_main(r):
        try:
            st = torch.cuda.Stream()
            with torch.cuda.stream(st):
                s = ipr.Solver(A_host, 2, phases, 1e-12, stream=st, world=world, rank=r, form=form,
                               local_group=grp, cert="crt")
                C = torch.empty_like(A_host).pin_memory()
                s.set_output(C)
                s.iterate(300)
                tr, out = s.trace(), s.outcome
                s.finalize(C)
                st.synchronize()
                res[r] = (out, tr, C.numpy().copy())
        except Exception as e:   # noqa: BLE001
            err[r] = e

    th = [threading.Thread(target=rank_main, args=(r,), daemon=True) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(600)
    ipr.ipr_test_local_group_destroy(grp)
    for e in err:
        if e is not None:
            raise e
    for out, tr, C in res:
        assert out == out1 == ipr.IPR_CONVERGED
        _same_trace(tr, tr1)
        np.testing.assert_array_equal(C, C1)
