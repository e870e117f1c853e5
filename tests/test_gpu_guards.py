"""Memory-safety check of every hot-path kernel in place of compute-sanitizer (closed on this pool,
profiles/r02_sanitizer.md): with guard bands behind every arena buffer (ipr_test_set_guards), solves of
every form, format and decomposition at ragged sizes must leave all bands intact -- an overrun past any
buffer end (mirror stores, residue planes, v bytes, CRT finish, panel exchanges) alters a band."""
import threading

import pytest

import synth

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
ipr = pytest.importorskip("paper_1703_02283_b200")

SCHEDULES = [
    ("symtri:fp8/cfp8>bf16>fp64crt@a/cbf16", 2), ("sym:fp8/cfp8>bf16>fp64crt@a/cbf16", 2),
    ("symtri:bf16>fp64oz@a/cbf16", 2), ("symtri:int8/cint8>bf16>fp64/cbf16", 2), ("sym:fp16>fp64/cbf16", 3),
    ("bf16>fp64", 2), ("tf32>fp64", 3), ("ns:tf32>fp64", 1), ("cpl:fp64", 2), ("fp64", 2),
]


@pytest.fixture(autouse=True)
def guards():
    ipr.ipr_test_set_guards(True)
    yield
    ipr.ipr_test_set_guards(False)


def _solve_checked(A, p, sched, **kw):
    import bench
    form, ph = bench.schedule(sched, A.shape[0])
    s = ipr.Solver(A, p, ph, 1e-12, form=form, **kw)
    s.iterate(200)
    bad = ipr.ipr_test_check_guards(s.ctx)
    out = s.outcome
    s.close()
    return bad, out


@pytest.mark.parametrize("n", [300, 520, 1000])
@pytest.mark.parametrize("sched,p", SCHEDULES, ids=[s[0] for s in SCHEDULES])
def test_guards_intact(n, sched, p):
    A = torch.from_numpy(synth.spd(n, 2.0, 40 + n)).cuda()
    bad, out = _solve_checked(A, p, sched)
    assert bad == -1, (sched, n, bad)
    assert out == ipr.IPR_CONVERGED


def test_guards_detect_an_overrun():
    A = torch.from_numpy(synth.spd(300, 2.0, 1)).cuda()
    s = ipr.Solver(A, 2, [ipr.make_phase("fp64")], 1e-12)
    s.iterate(3)
    assert ipr.ipr_test_check_guards(s.ctx) == -1
    assert ipr.ipr_test_check_guards(s.ctx, corrupt_first=True) == 0     # the positive control
    s.close()


@pytest.mark.parametrize("sched,grid", [("symtri:fp8/cfp8>bf16>fp64crt@a/cbf16", None), ("bf16>fp64", (2, 2))])
def test_guards_intact_sharded(sched, grid):
    import bench
    A = torch.from_numpy(synth.spd(1024, 2.0, 7)).cuda()
    form, ph = bench.schedule(sched, 1024)
    world = 4 if grid else 2
    grp = ipr.ipr_test_local_group_create(world)
    bad = [None] * world
    err = [None] * world

    def rank_main(r):
        try:
            st = torch.cuda.Stream()
            with torch.cuda.stream(st):
                s = ipr.Solver(A, 2, ph, 1e-12, stream=st, world=world, rank=r, form=form, local_group=grp, grid=grid)
                s.iterate(200)
                bad[r] = ipr.ipr_test_check_guards(s.ctx)
                s.close()
        except Exception as e:   # noqa: BLE001
            err[r] = e

    th = [threading.Thread(target=rank_main, args=(r,), daemon=True) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(600)
    ipr.ipr_test_local_group_destroy(grp)
    assert all(e is None for e in err), err
    assert bad == [-1] * world


@pytest.mark.parametrize("n", [300, 520, 1000])
@pytest.mark.parametrize("sched,p", [("symtri:fp8/cfp8>bf16>fp64crt@a/cbf16", 2), ("sym:bf16>fp64crt@a/cbf16", 2),
                                     ("sym:bf16>fp64crt@a/cbf16", 3)])
def test_guards_intact_crt_certificate(n, sched, p):
    # IPR_CERT_CRT (R-35): the grid-rounding split, the double-double finish with its mirrored hi / lo
    # stores, the double-double split and the certificate's statistics stay inside their buffers
    A = torch.from_numpy(synth.spd(n, 2.0, 60 + n)).cuda()
    bad, out = _solve_checked(A, p, sched, cert="crt")
    assert bad == -1, (sched, n, bad)
    assert out == ipr.IPR_CONVERGED
