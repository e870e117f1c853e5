"""World-size-2 CPU test (gloo) of the multi-GPU decomposition.

The CUDA engine shards every GEMM of the chain by output columns (rank g owns S_g), keeps Chat
replicated through an all-gather of per-rank panels, and reduces per-tile residual / delta
partials from GLOBAL slots.  This test drives that exact data flow on the CPU: the layout plan
comes from libipr's own host code (ipr_plan, no GPU needed), products are the oracle's column-
panel GEMM (same per-element k order as the full product), panels and partials travel through
torch.distributed all_gather over gloo.  It checks that
  * the ranks' plans tile the padded columns and the partial slots exactly once,
  * every iterate assembled from the 2 ranks' panels is bit-identical to the single-process
    oracle trajectory (Eq. 1), and
  * rho reduced in slot order is bit-identical for world = 1 and world = 2.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synth


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def emulate(A, p, iters, world, rank, m=52, gather=None):
    """Column-panel iteration in the library's layout; returns ([C_k], [rho_k])."""
    import paper_1703_02283_b200 as ipr
    n = A.shape[0]
    plan = ipr.ipr_plan(n, world, rank, ipr.IPR_FP64)
    npad, kp, col0 = plan["npad"], plan["kp"], plan["col0"]
    tm, tn, tiles_m, tiles_n = plan["tile_m"], plan["tile_n"], plan["tiles_m"], plan["tiles_n_total"]
    Ap = np.zeros((npad, npad)); Ap[:n, :n] = A
    n1, ninf, _ = oracle.norms(A)
    s = n1 * ninf
    ph = oracle.phase(oracle.FP64, mant_bits=m)
    cols = slice(col0, col0 + kp)

    def allgather_panels(panel):          # [npad][kp] local panel -> full row-major Chat
        if gather is None:
            return panel.copy()
        parts = gather(panel)
        return np.concatenate(parts, axis=1)

    def allgather_partials(local):        # local slots -> global slot array
        if gather is None:
            return local
        return np.concatenate(gather(local))

    C_panel = oracle.c0(Ap, s, ph)[:, cols]        # C_0 of the padded matrix, local panel
    hist, rhos = [], []
    for k in range(iters):
        C = allgather_panels(C_panel)              # replicated Chat (FP64 phase: = container)
        hist.append(C[:n, :n].copy())
        X = Ap
        T = np.zeros((npad, npad))
        for j in range(p):
            T = np.zeros((npad, npad))
            oracle.gemm_cols(C, X, T, col0, col0 + kp)
            X = T
        # per-tile residual partials in global slots [tn_global][tm]
        I = np.eye(npad)[:, cols]
        D = (I - T[:, cols])
        D[n:, :] = 0.0
        if col0 + kp > n:
            D[:, max(0, n - col0):] = 0.0
        local = np.zeros((kp // tn) * tiles_m)
        for a in range(kp // tn):
            for b in range(tiles_m):
                blk = D[b * tm:(b + 1) * tm, a * tn:(a + 1) * tn]
                local[a * tiles_m + b] = np.sum(blk * blk)
        part = allgather_partials(local)
        assert part.size == tiles_m * tiles_n
        rho = 0.0
        for v in part:
            rho += v
        rhos.append(np.sqrt(rho))
        P = np.zeros((npad, npad))
        oracle.gemm_cols(C, T, P, col0, col0 + kp)
        a_ = float(p + 1) * C_panel
        d_ = a_ - P[:, cols]
        e_ = d_ / float(p)
        C_panel = oracle.qm(e_, 11, m)
    return hist, rhos


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1703_02283_b200 as ipr
        A = synth.spd(300, 2.0, 21)

        def gather(arr):
            t = torch.from_numpy(np.ascontiguousarray(arr))
            out = [torch.empty_like(t) for _ in range(world)]
            dist.all_gather(out, t)
            return [o.numpy() for o in out]

        plans = [None] * world
        dist.all_gather_object(plans, ipr.ipr_plan(300, world, rank, ipr.IPR_FP64))
        hist, rhos = emulate(A, 2, 6, world, rank, gather=gather)
        if rank == 0:
            q.put(("ok", plans, hist, rhos))
    except Exception as e:  # surface the failure to the parent
        if rank == 0:
            q.put(("err", repr(e), None, None))
        raise
    finally:
        dist.destroy_process_group()


def test_plan_covers_columns_and_slots():
    import paper_1703_02283_b200 as ipr
    for n in [64, 300, 1024, 8192, 32768]:
        for world in [1, 2, 4, 8]:
            for prec in [ipr.IPR_FP64, ipr.IPR_BF16]:
                plans = [ipr.ipr_plan(n, world, r, prec) for r in range(world)]
                npad = plans[0]["npad"]
                assert npad >= n and npad % (256 * world) == 0
                cols = np.zeros(npad, int)
                for pl in plans:
                    assert pl["npad"] == npad and pl["kp"] * world == npad
                    cols[pl["col0"]:pl["col0"] + pl["kp"]] += 1
                    assert pl["kp"] % pl["tile_n"] == 0
                assert np.all(cols == 1)
                slots = [pl["part0"] for pl in plans] + [pl["tiles_m"] * pl["tiles_n_total"] for pl in plans[:1]]
                per = plans[0]["kp"] // plans[0]["tile_n"] * plans[0]["tiles_m"]
                assert all(slots[r] == r * per for r in range(world))
    assert ipr.ipr_plan(32768, 8, 7, ipr.IPR_BF16)["kp"] == 4096


def test_world2_gloo_matches_single_rank_and_oracle():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    status, plans, hist2, rhos2 = q.get(timeout=300)
    for pr in procs:
        pr.join(timeout=300)
    assert status == "ok", plans
    assert all(pr.exitcode == 0 for pr in procs)
    assert plans[0]["col0"] == 0 and plans[1]["col0"] == plans[0]["kp"]
    A = synth.spd(300, 2.0, 21)
    hist1, rhos1 = emulate(A, 2, 6, 1, 0)
    r = oracle.solve(A, 2, [oracle.phase()], 0.0, 6, hist=6)
    for k in range(6):
        np.testing.assert_array_equal(hist2[k], hist1[k])
        np.testing.assert_array_equal(hist2[k], r.C_hist[k])
    assert rhos2 == rhos1                     # bit-identical slot-ordered reduction
    np.testing.assert_allclose(rhos1, r.rho, rtol=1e-13)


def emulate_sym(A, iters, world, rank, gather=None):
    """The symmetric form's (R-22, p = 2, FP64) column-panel data flow of the engine at G > 1:
    Z_1[:, S_g] = A C[:, S_g] (A operand: the full Ahat), Z_2[:, S_g] = C Z_1[:, S_g], R = I - Z_2,
    W[:, S_g] = C R[:, S_g]; W panels all-gathered (the W + W^T update needs W(j, i) from the
    other ranks' panels), C_{k+1}[:, S_g] = C + (W + W^T)/4, C panels all-gathered."""
    import paper_1703_02283_b200 as ipr
    n = A.shape[0]
    plan = ipr.ipr_plan(n, world, rank, ipr.IPR_FP64)
    npad, kp, col0 = plan["npad"], plan["kp"], plan["col0"]
    Ap = np.zeros((npad, npad)); Ap[:n, :n] = A
    n1, ninf, _ = oracle.norms(A)
    cols = slice(col0, col0 + kp)

    def full(panel):
        return panel.copy() if gather is None else np.concatenate(gather(panel), axis=1)

    C_panel = oracle.c0(Ap, n1 * ninf, oracle.phase())[:, cols]
    hist = []
    for k in range(iters):
        C = full(C_panel)
        hist.append(C[:n, :n].copy())
        Z1 = np.zeros((npad, npad)); oracle.gemm_cols(Ap, C, Z1, col0, col0 + kp)
        Z2 = np.zeros((npad, npad)); oracle.gemm_cols(C, Z1, Z2, col0, col0 + kp)
        R = np.zeros((npad, npad))
        R[:, cols] = np.eye(npad)[:, cols] - Z2[:, cols]
        R[n:, :] = 0.0
        R[:, n:] = 0.0
        W = np.zeros((npad, npad)); oracle.gemm_cols(C, R, W, col0, col0 + kp)
        Wf = full(W[:, cols])
        C_panel = C_panel + (Wf[:, cols] + Wf.T[:, cols]) / 4.0
    return hist


def _worker_sym(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        A = synth.spd(300, 2.0, 22)

        def gather(arr):
            t = torch.from_numpy(np.ascontiguousarray(arr))
            out = [torch.empty_like(t) for _ in range(world)]
            dist.all_gather(out, t)
            return [o.numpy() for o in out]

        hist = emulate_sym(A, 5, world, rank, gather=gather)
        if rank == 0:
            q.put(("ok", hist))
    except Exception as e:
        if rank == 0:
            q.put(("err", repr(e)))
        raise
    finally:
        dist.destroy_process_group()


def test_world2_gloo_symmetric_form_matches_oracle():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_sym, args=(r, 2, port, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    status, hist2 = q.get(timeout=300)
    for pr in procs:
        pr.join(timeout=300)
    assert status == "ok", hist2
    assert all(pr.exitcode == 0 for pr in procs)
    A = synth.spd(300, 2.0, 22)
    hist1 = emulate_sym(A, 5, 1, 0)
    r = oracle.solve(A, 2, [oracle.phase()], 0.0, 5, hist=5, form=oracle.FORM_SYMMETRIC)
    for k in range(5):
        np.testing.assert_array_equal(hist2[k], hist1[k])
        np.testing.assert_array_equal(hist2[k], r.C_hist[k])     # bit-identical to the oracle
        assert np.array_equal(hist2[k], hist2[k].T)


def emulate_2d(A, p, iters, grows, gcols, rank, row_gather=None, col_gather=None, all_gather=None, tm=128, tn=256):
    """The 2-D P_r x P_c grid's data flow of the engine (literal form, FP64): rank
    (r, c) owns the block (R_r, S_c) of C and of every T_j; Chat row panels gather along the grid row,
    T_{j-1} column panels along the grid column before every GEMM, each residual partial is taken
    from the rank owning its tile (global slot order tn * tiles_m + tm, as k_select_partials)."""
    n = A.shape[0]
    world = grows * gcols
    unit = 256 * world
    npad = (n + unit - 1) // unit * unit
    mr, kp = npad // grows, npad // gcols
    r, c = rank // gcols, rank % gcols
    rows, cols = slice(r * mr, (r + 1) * mr), slice(c * kp, (c + 1) * kp)
    tiles_m, tiles_n = npad // tm, npad // tn
    Ap = np.zeros((npad, npad)); Ap[:n, :n] = A
    n1, ninf, _ = oracle.norms(A)
    ph = oracle.phase(oracle.FP64)
    C_blk = oracle.c0(Ap, n1 * ninf, ph)[rows, cols]

    def row_panel(blk):          # C[R_r, :] from the grid row's blocks, in grid-column order
        return blk.copy() if row_gather is None else np.concatenate(row_gather(blk), axis=1)

    def col_panel(blk):          # T[:, S_c] from the grid column's blocks, in grid-row order
        return blk.copy() if col_gather is None else np.concatenate(col_gather(blk), axis=0)

    def block_product(Cr, X):    # (C X)[R_r, S_c] with the oracle's per-element k order
        Cf = np.zeros((npad, npad)); Cf[rows, :] = Cr
        Xf = np.zeros((npad, npad)); Xf[:, cols] = X
        Z = np.zeros((npad, npad)); oracle.gemm_cols(Cf, Xf, Z, c * kp, (c + 1) * kp)
        return Z[rows, cols]

    hist, rhos = [], []
    for k in range(iters):
        Cr = row_panel(C_blk)
        X = Ap[:, cols]
        for j in range(p):
            T_blk = block_product(Cr, X)
            X = col_panel(T_blk)
        # residual partials of this rank's tiles at their GLOBAL slots
        I = np.eye(npad)[rows, cols]
        D = I - T_blk
        gi = np.arange(r * mr, (r + 1) * mr)[:, None]
        gj = np.arange(c * kp, (c + 1) * kp)[None, :]
        D = np.where((gi < n) & (gj < n), D, 0.0)
        part = np.zeros(tiles_m * tiles_n)
        for a in range(kp // tn):
            for b in range(mr // tm):
                blk = D[b * tm:(b + 1) * tm, a * tn:(a + 1) * tn]
                part[(c * kp // tn + a) * tiles_m + r * mr // tm + b] = np.sum(blk * blk)
        parts = [part] if all_gather is None else all_gather(part)
        sel = np.empty_like(part)
        for sl in range(part.size):
            tnn, tmm = sl // tiles_m, sl % tiles_m
            owner = ((tmm * tm) // mr) * gcols + (tnn * tn) // kp
            sel[sl] = parts[owner][sl]
        rho = 0.0
        for v in sel:
            rho += v
        rhos.append(np.sqrt(rho))
        P_blk = block_product(Cr, X)
        C_blk = oracle.qm((float(p + 1) * C_blk - P_blk) / float(p), 11, 52)
        blocks = [C_blk] if all_gather is None else all_gather(C_blk)
        hist.append(blocks)
    return hist, rhos, (npad, mr, kp)


def _worker_2d(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        A = synth.spd(300, 2.0, 23)
        row_groups = [dist.new_group([0, 1]), dist.new_group([2, 3])]
        col_groups = [dist.new_group([0, 2]), dist.new_group([1, 3])]

        def gatherer(group, size):
            def g(arr):
                t = torch.from_numpy(np.ascontiguousarray(arr))
                out = [torch.empty_like(t) for _ in range(size)]
                dist.all_gather(out, t, group=group)
                return [o.numpy() for o in out]
            return g

        hist, rhos, dims = emulate_2d(A, 2, 4, 2, 2, rank, row_gather=gatherer(row_groups[rank // 2], 2),
                                      col_gather=gatherer(col_groups[rank % 2], 2), all_gather=gatherer(None, 4))
        if rank == 0:
            q.put(("ok", hist, rhos, dims))
    except Exception as e:
        if rank == 0:
            q.put(("err", repr(e), None, None))
        raise
    finally:
        dist.destroy_process_group()


def test_world4_gloo_2d_grid_matches_oracle():
    # the 2 x 2 grid option: every iterate assembled from the four blocks is bit-identical to the
    # single-process oracle trajectory of Eq. (1), and rho reduced from owner-selected partials in slot
    # order equals the one-rank value bit for bit
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_2d, args=(r, 4, port, q)) for r in range(4)]
    for pr in procs:
        pr.start()
    status, hist, rhos, dims = q.get(timeout=600)
    for pr in procs:
        pr.join(timeout=300)
    assert status == "ok", hist
    assert all(pr.exitcode == 0 for pr in procs)
    npad, mr, kp = dims
    A = synth.spd(300, 2.0, 23)
    r = oracle.solve(A, 2, [oracle.phase()], 0.0, 5, hist=5)
    hist1, rhos1, _ = emulate_2d(A, 2, 4, 1, 1, 0, all_gather=lambda a: [a])
    for k in range(4):
        full = np.zeros((npad, npad))
        for rank, blk in enumerate(hist[k]):
            rr, cc = rank // 2, rank % 2
            full[rr * mr:(rr + 1) * mr, cc * kp:(cc + 1) * kp] = blk
        np.testing.assert_array_equal(full[:300, :300], r.C_hist[k + 1])
        np.testing.assert_array_equal(full[:300, :300], hist1[k][0][:300, :300])
    assert rhos == rhos1
    np.testing.assert_allclose(rhos, r.rho[:4], rtol=1e-13)
