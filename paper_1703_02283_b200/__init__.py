"""B200-native (sm_100a) inverse matrix p-th roots -- the Bini iteration of arXiv:1703.02283.

Thin Python binding of libipr.so (include/ipr.h): argument marshalling only.  Every step of
the hot path (norms, C_0, the p+1 GEMMs, the fused residual/update epilogues, reductions,
conversions, all-gathers) runs in the library's CUDA kernels.  There is no CPU fallback:
importing this package without the built library raises, and every call that the GPU path
cannot serve returns an error status.

PyTorch is used only for device memory and streams (pass tensors or raw device pointers).
"""
from __future__ import annotations

import ctypes as C
import math
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "lib", "libipr.so")

IPR_OK, IPR_E_INVALID_ARG, IPR_E_NOT_SYMMETRIC, IPR_E_STATE = 0, 1, 2, 3
IPR_E_UNSUPPORTED, IPR_E_OOM, IPR_E_CUDA, IPR_E_NCCL = 4, 5, 6, 7
IPR_FP64, IPR_TF32, IPR_BF16, IPR_FP16, IPR_FP8, IPR_INT8, IPR_FP64_OZ, IPR_FP64_CRT = 0, 1, 2, 3, 4, 5, 6, 7
IPR_RNE, IPR_RTZ = 0, 1
IPR_MANT_ADAPTIVE = -2   # IPR_FP64_OZ / IPR_FP64_CRT phases: Ozaki digits / stored bits chosen per iteration (R-26)
IPR_RUNNING, IPR_CONVERGED, IPR_ITER_LIMIT, IPR_DIVERGED, IPR_NONFINITE = 0, 1, 2, 3, 4
IPR_DEC_CONTINUE, IPR_DEC_SWITCH = 0, 5
PREC_NAMES = {IPR_FP64: "fp64", IPR_TF32: "tf32", IPR_BF16: "bf16", IPR_FP16: "fp16", IPR_FP8: "fp8",
              IPR_INT8: "int8", IPR_FP64_OZ: "fp64oz", IPR_FP64_CRT: "fp64crt"}
PREC_BY_NAME = {v: k for k, v in PREC_NAMES.items()}
OUTCOME_NAMES = {0: "running", 1: "converged", 2: "iter_limit", 3: "diverged", 4: "nonfinite"}

# Every symbol include/ipr.h and include/ipr_testing.h declare.
EXPORTED = ["ipr_init", "ipr_set_schedule", "ipr_iterate", "ipr_residual", "ipr_get_trace",
            "ipr_get_iterate", "ipr_get_norms", "ipr_finalize", "ipr_last_error",
            "ipr_nccl_unique_id", "ipr_version", "ipr_test_quantize", "ipr_test_gemm",
            "ipr_launch_count", "ipr_plan", "ipr_set_form", "ipr_bench_gemm", "ipr_bench_gemm_epi",
            "ipr_test_set_digits", "ipr_test_crt_table", "ipr_set_cert", "ipr_test_peek",
            "ipr_test_local_group_create", "ipr_test_local_group_destroy", "ipr_test_init_local",
            "ipr_test_set_guards", "ipr_test_check_guards", "ipr_set_output", "ipr_test_crt_signed", "ipr_test_nccl_selftest",
            "ipr_test_cert_info"]
IPR_FORM_LITERAL, IPR_FORM_NEWTON_SCHULZ, IPR_FORM_SYMMETRIC, IPR_FORM_SYMMETRIC_TRI, IPR_FORM_COUPLED = 0, 1, 2, 3, 4
IPR_FORM_SYMMETRIC_TRIZ = 5   # reading R-37
IPR_CERT_FP64, IPR_CERT_PHASE, IPR_CERT_FP64_CHAIN, IPR_CERT_CRT = 0, 1, 2, 3
CERT_BY_NAME = {"fp64": IPR_CERT_FP64, "dmma": IPR_CERT_FP64, "phase": IPR_CERT_PHASE,
                "fp64chain": IPR_CERT_FP64_CHAIN, "crt": IPR_CERT_CRT}
FORM_BY_NAME = {"literal": IPR_FORM_LITERAL, "newton_schulz": IPR_FORM_NEWTON_SCHULZ, "ns": IPR_FORM_NEWTON_SCHULZ,
                "symmetric": IPR_FORM_SYMMETRIC, "sym": IPR_FORM_SYMMETRIC,
                "symmetric_tri": IPR_FORM_SYMMETRIC_TRI, "symtri": IPR_FORM_SYMMETRIC_TRI,
                "symmetric_triz": IPR_FORM_SYMMETRIC_TRIZ, "symtriz": IPR_FORM_SYMMETRIC_TRIZ,
                "coupled": IPR_FORM_COUPLED}


class IprError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"ipr status {status}: {msg}")
        self.status = status


class ipr_phase(C.Structure):
    _fields_ = [("prec", C.c_int), ("mant_bits", C.c_int), ("round", C.c_int),
                ("switch_tol", C.c_double), ("plateau_ratio", C.c_double),
                ("plateau_arm", C.c_double), ("max_iters", C.c_int), ("corr_prec", C.c_int)]


class ipr_record(C.Structure):
    _fields_ = [("k", C.c_int), ("phase", C.c_int), ("prec", C.c_int), ("mant_bits", C.c_int),
                ("decision", C.c_int), ("rho", C.c_double), ("rho_hat", C.c_double),
                ("delta", C.c_double), ("gemm_ms", C.c_double), ("upd_ms", C.c_double),
                ("digits", C.c_int), ("rho_cert", C.c_double), ("moduli", C.c_int),
                ("ztri", C.c_int), ("kern_ms", C.c_double), ("gap_ms", C.c_double)]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is not built: run `python -c 'import __graft_entry__ as g; "
                          "g.build()'` (no CPU fallback exists)")
    L = C.CDLL(LIB_PATH, mode=C.RTLD_GLOBAL)
    vp, i64, dp = C.c_void_p, C.c_int64, C.POINTER(C.c_double)
    L.ipr_init.argtypes = [C.POINTER(vp), i64, vp, i64, vp, C.c_int, C.c_int, vp, C.c_int, C.c_int]
    L.ipr_set_schedule.argtypes = [vp, C.c_int, C.POINTER(ipr_phase), C.c_int, C.c_double]
    L.ipr_iterate.argtypes = [vp, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int)]
    L.ipr_residual.argtypes = [vp, C.c_int, dp]
    L.ipr_get_trace.argtypes = [vp, C.POINTER(ipr_record), C.c_int, C.POINTER(C.c_int)]
    L.ipr_get_iterate.argtypes = [vp, C.c_int, vp, i64]
    L.ipr_get_norms.argtypes = [vp, dp]
    L.ipr_finalize.argtypes = [vp, vp, i64]
    L.ipr_set_output.argtypes = [vp, vp, i64]
    L.ipr_last_error.argtypes = [vp]
    L.ipr_last_error.restype = C.c_char_p
    L.ipr_nccl_unique_id.argtypes = [vp]
    L.ipr_version.restype = C.c_char_p
    L.ipr_test_quantize.argtypes = [C.c_int, vp, vp, i64, C.c_int, C.c_int, C.c_int, vp]
    L.ipr_test_gemm.argtypes = [C.c_int, i64, vp, vp, vp, vp]
    L.ipr_launch_count.restype = C.c_int64
    L.ipr_plan.argtypes = [i64, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_int64)]
    L.ipr_set_form.argtypes = [vp, C.c_int]
    L.ipr_set_cert.argtypes = [vp, C.c_int]
    L.ipr_test_peek.argtypes = [vp, C.c_int, vp, C.POINTER(C.c_int64)]
    L.ipr_test_cert_info.argtypes = [vp, C.POINTER(C.c_double)]
    L.ipr_test_local_group_create.argtypes = [C.c_int, C.POINTER(vp)]
    L.ipr_test_local_group_destroy.argtypes = [vp]
    L.ipr_test_set_guards.argtypes = [C.c_int]
    L.ipr_test_check_guards.argtypes = [vp, C.c_int, C.POINTER(C.c_int)]
    L.ipr_test_init_local.argtypes = [C.POINTER(vp), i64, vp, i64, vp, vp, C.c_int, C.c_int, C.c_int]
    L.ipr_bench_gemm.argtypes = [C.c_int, i64, C.c_int, C.c_int, vp, dp]
    L.ipr_bench_gemm_epi.argtypes = [C.c_int, i64, C.c_int, C.c_int, C.c_int, vp, dp]
    L.ipr_test_set_digits.argtypes = [C.c_int]
    L.ipr_test_crt_signed.argtypes = [C.c_int]
    L.ipr_test_crt_table.argtypes = [C.c_int, C.c_int, i64, C.POINTER(C.c_int), dp, C.POINTER(C.c_int), C.POINTER(C.c_int)]
    for f in EXPORTED:
        if f not in ("ipr_last_error", "ipr_version", "ipr_launch_count"):
            getattr(L, f).restype = C.c_int
    return L


_lib = _load()


def lib():
    return _lib


def _ptr(x) -> int:
    """Device pointer of a torch tensor (or an int/None passed through)."""
    if x is None:
        return None
    if isinstance(x, int):
        return x
    return x.data_ptr()


def _check_matrix(x, n: int, what: str, ref=None, host_ok: bool = False):
    """A boundary matrix must be an FP64 tensor, n x n, unit column stride (ipr.h: FP64, row-major,
    leading dimension >= n), on the device -- or in host memory where the call takes one (host_ok:
    ipr_init's A, ipr_finalize's / ipr_set_output's / ipr_get_iterate's C) -- anything else would make
    the library read or write the wrong bytes.  Raw integer pointers are passed through unchecked."""
    if x is None or isinstance(x, int):
        return
    import torch
    if x.dtype != torch.float64:
        raise ValueError(f"{what}: dtype must be torch.float64 (got {x.dtype})")
    if not x.is_cuda and not (host_ok and x.device.type == "cpu"):
        raise ValueError(f"{what}: must be a CUDA tensor (got device {x.device})")
    if (ref is not None and not isinstance(ref, int) and x.is_cuda and ref.is_cuda
            and x.device != ref.device):
        raise ValueError(f"{what}: on {x.device}, A is on {ref.device}")
    if x.dim() != 2 or x.shape[0] < n or x.shape[1] < n:
        raise ValueError(f"{what}: shape must be ({n}, {n}) (got {tuple(x.shape)})")
    if x.stride(1) != 1 or x.stride(0) < n:
        raise ValueError(f"{what}: needs stride(1) == 1 and stride(0) >= n (got {x.stride()})")


def _stream(s) -> int:
    if s is None:
        return None
    if isinstance(s, int):
        return s
    return s.cuda_stream


def _check(st: int, ctx=None):
    if st != IPR_OK:
        msg = _lib.ipr_last_error(ctx)
        raise IprError(st, msg.decode() if msg else "")


# ---- the C-ABI, same names ------------------------------------------------------------------
def ipr_version() -> str:
    return _lib.ipr_version().decode()


def ipr_last_error(ctx=None) -> str:
    m = _lib.ipr_last_error(ctx)
    return m.decode() if m else ""


def ipr_nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _check(_lib.ipr_nccl_unique_id(buf))
    return buf.raw


def ipr_init(n: int, A, lda: int | None = None, stream=None, world: int = 1, rank: int = 0,
             nccl_unique_id: bytes | None = None, grid_rows: int = 1, grid_cols: int | None = None):
    _check_matrix(A, n, "ipr_init: A", host_ok=True)
    ctx = C.c_void_p()
    uid = C.create_string_buffer(nccl_unique_id, 128) if nccl_unique_id is not None else None
    _check(_lib.ipr_init(C.byref(ctx), n, _ptr(A), lda if lda is not None else n, _stream(stream),
                         world, rank, uid, grid_rows, grid_cols if grid_cols is not None else world))
    return ctx


def ipr_test_local_group_create(world: int):
    """An in-process group of `world` ranks on the current device (ipr_testing.h)."""
    g = C.c_void_p()
    _check(_lib.ipr_test_local_group_create(world, C.byref(g)))
    return g


def ipr_test_local_group_destroy(group):
    _check(_lib.ipr_test_local_group_destroy(group))


def ipr_test_init_local(n: int, A, lda: int | None, stream, group, rank: int, grid_rows: int = 1,
                        grid_cols: int | None = None, world: int | None = None):
    """ipr_init for rank `rank` of a local group (call from the rank's own host thread)."""
    _check_matrix(A, n, "ipr_test_init_local: A", host_ok=True)
    ctx = C.c_void_p()
    _check(_lib.ipr_test_init_local(C.byref(ctx), n, _ptr(A), lda if lda is not None else n, _stream(stream),
                                    group, rank, grid_rows, grid_cols if grid_cols is not None else world))
    return ctx


def make_phase(prec="fp64", mant_bits=-1, round="rne", switch_tol=0.0, plateau_ratio=0.0,
               plateau_arm=0.5, max_iters=0, corr_prec=-1) -> ipr_phase:
    pr = PREC_BY_NAME[prec] if isinstance(prec, str) else int(prec)
    rd = {"rne": IPR_RNE, "rtz": IPR_RTZ}[round] if isinstance(round, str) else int(round)
    cp = PREC_BY_NAME[corr_prec] if isinstance(corr_prec, str) else int(corr_prec)
    return ipr_phase(pr, mant_bits, rd, switch_tol, plateau_ratio, plateau_arm, max_iters, cp)


def ipr_set_schedule(ctx, p: int, phases, final_tol: float):
    arr = (ipr_phase * len(phases))(*phases)
    _check(_lib.ipr_set_schedule(ctx, p, arr, len(phases), final_tol), ctx)


def ipr_set_form(ctx, form):
    f = FORM_BY_NAME[form] if isinstance(form, str) else int(form)
    _check(_lib.ipr_set_form(ctx, f), ctx)


def ipr_set_cert(ctx, mode):
    m = CERT_BY_NAME[mode] if isinstance(mode, str) else int(mode)
    _check(_lib.ipr_set_cert(ctx, m), ctx)


def ipr_iterate(ctx, max_iters: int):
    done, out = C.c_int(0), C.c_int(0)
    _check(_lib.ipr_iterate(ctx, max_iters, C.byref(done), C.byref(out)), ctx)
    return done.value, out.value


def ipr_residual(ctx, certify: int = 0) -> float:
    """certify: 0 the in-chain residual, 1 the context's certificate of the best iterate, 2 its FP64 DMMA
    evaluation (ipr.h)."""
    r = C.c_double(0)
    _check(_lib.ipr_residual(ctx, int(certify), C.byref(r)), ctx)
    return r.value


def ipr_get_trace(ctx):
    cnt = C.c_int(0)
    _check(_lib.ipr_get_trace(ctx, None, 0, C.byref(cnt)), ctx)
    buf = (ipr_record * max(cnt.value, 1))()
    _check(_lib.ipr_get_trace(ctx, buf, cnt.value, C.byref(cnt)), ctx)
    return [dict(k=r.k, phase=r.phase, prec=PREC_NAMES[r.prec], mant_bits=r.mant_bits,
                 decision=r.decision, rho=r.rho, rho_hat=r.rho_hat, delta=r.delta, gemm_ms=r.gemm_ms,
                 upd_ms=r.upd_ms, digits=r.digits, rho_cert=r.rho_cert, moduli=r.moduli, ztri=r.ztri, kern_ms=r.kern_ms,
                 gap_ms=r.gap_ms)
            for r in buf[:cnt.value]]


def ipr_get_iterate(ctx, which: int, C_out, ldc: int | None = None):
    if C_out is not None and not isinstance(C_out, int):
        _check_matrix(C_out, C_out.shape[0], "ipr_get_iterate: C_out", host_ok=True)
    _check(_lib.ipr_get_iterate(ctx, which, _ptr(C_out), ldc if ldc is not None else C_out.shape[1]), ctx)


def ipr_get_norms(ctx):
    out = (C.c_double * 4)()
    _check(_lib.ipr_get_norms(ctx, out), ctx)
    return tuple(out)


def ipr_set_output(ctx, C_out=None, ldc: int | None = None):
    """The destination ipr_finalize will get (host or device): the certified answer streams there early."""
    _check_matrix(C_out, C_out.shape[0] if C_out is not None and not isinstance(C_out, int) else 0,
                  "ipr_set_output: C_out", host_ok=True)
    ld = ldc if ldc is not None else (C_out.stride(0) if C_out is not None and not isinstance(C_out, int) else 0)
    _check(_lib.ipr_set_output(ctx, _ptr(C_out), ld), ctx)


def ipr_finalize(ctx, C_out=None, ldc: int | None = None):
    if C_out is not None and not isinstance(C_out, int):
        try:
            _check_matrix(C_out, C_out.shape[0], "ipr_finalize: C_out", host_ok=True)
        except ValueError:
            _lib.ipr_finalize(ctx, None, 0)   # still free the context
            raise
    st = _lib.ipr_finalize(ctx, _ptr(C_out), ldc if ldc is not None else (C_out.shape[1] if C_out is not None else 0))
    _check(st)


def ipr_test_quantize(mode: int, x_in, x_out, m: int = 0, round: int = IPR_RNE, sigma: int = 0, stream=None):
    _check(_lib.ipr_test_quantize(mode, _ptr(x_in), _ptr(x_out), x_in.numel(), m, round, sigma, _stream(stream)))


def ipr_test_gemm(prec: int, n: int, X, Yt, Z, stream=None):
    _check(_lib.ipr_test_gemm(prec, n, _ptr(X), _ptr(Yt), _ptr(Z), _stream(stream)))


def ipr_test_nccl_selftest():
    """NCCL transport plumbing on one GPU (ipr_testing.h); raises IprError on failure."""
    _check(_lib.ipr_test_nccl_selftest())


def ipr_test_crt_signed(on: bool):
    """Force the symmetric CRT residue convention (s8 x s8) at every K (ipr_testing.h)."""
    _check(_lib.ipr_test_crt_signed(1 if on else 0))


def ipr_test_set_digits(digits: int):
    """Ozaki digits S (OZ) / bits b = min(53, 7 S) (CRT) of ipr_test_gemm / ipr_bench_gemm products."""
    _check(_lib.ipr_test_set_digits(digits))


def ipr_test_crt_table(N: int, b: int = 53, n: int = 8192) -> dict:
    """Host-side CRT constants of N moduli (no GPU): moduli, inverses, sliced weights; n_for = the
    moduli a product with b bits at order n uses; b_for = the bits of S = b Ozaki-equivalent digits."""
    iv = (C.c_int * 40)()
    dv = (C.c_double * 64)()
    nf, bf = C.c_int(0), C.c_int(0)
    _check(_lib.ipr_test_crt_table(N, b, n, iv, dv, C.byref(nf), C.byref(bf)))
    return dict(moduli=list(iv[:N]), inv=list(iv[20:20 + N]),
                HLR=[tuple(dv[3 * l:3 * l + 3]) for l in range(N)], M_HLR=tuple(dv[54:57]),
                p2s=(dv[57], dv[58]), n_for=nf.value, b_for=bf.value)


def ipr_bench_gemm(prec, n: int, warmup: int = 2, iters: int = 5, stream=None) -> float:
    """Average device ms of the hot-path GEMM kernel of a format at order n (2 n^3 flop)."""
    pr = PREC_BY_NAME[prec] if isinstance(prec, str) else int(prec)
    ms = C.c_double(0)
    _check(_lib.ipr_bench_gemm(pr, n, warmup, iters, _stream(stream), C.byref(ms)))
    return ms.value


def ipr_bench_gemm_epi(prec, n: int, warmup: int = 2, iters: int = 5, epi: int = 0, stream=None) -> float:
    """ipr_bench_gemm with an explicit epilogue (0 default, 1 none, 2 STORE_T, 3 TSCRATCH)."""
    pr = PREC_BY_NAME[prec] if isinstance(prec, str) else int(prec)
    ms = C.c_double(0)
    _check(_lib.ipr_bench_gemm_epi(pr, n, warmup, iters, epi, _stream(stream), C.byref(ms)))
    return ms.value


IPR_PEEK_AHAT, IPR_PEEK_CHAT, IPR_PEEK_Z1, IPR_PEEK_RHAT, IPR_PEEK_W, IPR_PEEK_CHATC = 0, 1, 2, 3, 4, 5


CERT_INFO_KEYS = ("bound", "est", "beta", "dY", "dA", "A2", "Y2", "eY", "eP", "moduli")


def ipr_test_cert_info(ctx) -> dict:
    """The terms of the last IPR_CERT_CRT certificate (reading R-35; ipr_testing.h)."""
    out = (C.c_double * 10)()
    _check(_lib.ipr_test_cert_info(ctx, out), ctx)
    return dict(zip(CERT_INFO_KEYS, list(out)))


def ipr_test_peek(ctx, what: int, npad: int):
    """An intermediate of the last step as an (npad, npad) FP64 CUDA tensor (raw buffer order; see
    ipr_testing.h for which are K-major)."""
    import torch
    out = torch.empty((npad, npad), dtype=torch.float64, device="cuda")
    got = C.c_int64(0)
    _check(_lib.ipr_test_peek(ctx, what, _ptr(out), C.byref(got)), ctx)
    if got.value != npad:
        raise IprError(IPR_E_INVALID_ARG, f"ipr_test_peek: npad is {got.value}, not {npad}")
    return out


def ipr_test_set_guards(on: bool):
    _check(_lib.ipr_test_set_guards(int(on)))


def ipr_test_check_guards(ctx, corrupt_first: bool = False) -> int:
    """Index of the first altered arena guard band, -1 if all are intact (ipr_testing.h)."""
    bad = C.c_int(0)
    _check(_lib.ipr_test_check_guards(ctx, int(corrupt_first), C.byref(bad)), ctx)
    return bad.value


def ipr_launch_count() -> int:
    return _lib.ipr_launch_count()


def ipr_plan(n: int, world: int, rank: int, prec: int = IPR_FP64) -> dict:
    """Host-side layout plan of the 1 x world column-panel decomposition (no GPU needed)."""
    out = (C.c_int64 * 8)()
    _check(_lib.ipr_plan(n, world, rank, prec, out))
    keys = ["npad", "kp", "col0", "tile_m", "tile_n", "tiles_m", "tiles_n_total", "part0"]
    return dict(zip(keys, list(out)))


# ---- convenience wrapper (still marshalling only) -------------------------------------------
class Solver:
    """Owns one ipr_ctx.  A: FP64 CUDA tensor (n x n, symmetric), kept alive by the Solver."""

    def __init__(self, A, p: int, phases, final_tol: float = 1e-12, stream=None, world: int = 1,
                 rank: int = 0, nccl_unique_id: bytes | None = None, form="literal", cert="fp64",
                 local_group=None, grid=None):
        _check_matrix(A, A.shape[0], "Solver: A", host_ok=True)
        self.A = A
        self.n = A.shape[0]
        gr, gc = grid if grid is not None else (1, world)
        if local_group is not None:   # test transport: in-process ranks on one device (ipr_testing.h)
            self.ctx = ipr_test_init_local(self.n, A, A.stride(0), stream, local_group, rank, gr, gc)
        else:
            self.ctx = ipr_init(self.n, A, A.stride(0), stream, world, rank, nccl_unique_id, gr, gc)
        try:
            ipr_set_schedule(self.ctx, p, [ph if isinstance(ph, ipr_phase) else make_phase(**ph)
                                           for ph in phases], final_tol)
            ipr_set_form(self.ctx, form)
            ipr_set_cert(self.ctx, cert)
        except Exception:
            ipr_finalize(self.ctx)
            self.ctx = None
            raise
        self.outcome = IPR_RUNNING
        self.iters = 0

    def iterate(self, max_iters: int = 1000) -> int:
        done, out = ipr_iterate(self.ctx, max_iters)
        self.iters += done
        self.outcome = out
        return out

    def trace(self):
        return ipr_get_trace(self.ctx)

    def residual(self, certify: int = 0) -> float:
        return ipr_residual(self.ctx, certify)

    def norms(self):
        return ipr_get_norms(self.ctx)

    def iterate_copy(self, which: int = 0, out=None):
        import torch
        if out is None:
            out = torch.empty((self.n, self.n), dtype=torch.float64, device=self.A.device)
        _check_matrix(out, self.n, "iterate_copy: out", self.A, host_ok=True)
        ipr_get_iterate(self.ctx, which, out, out.stride(0))
        return out

    def set_output(self, out):
        """Register ipr_finalize's destination (ipr_set_output): the certified answer streams there
        while its FP64 certificate runs."""
        _check_matrix(out, self.n, "set_output: out", self.A, host_ok=True)
        ipr_set_output(self.ctx, out, out.stride(0))
        self._out = out

    def finalize(self, out=None):
        import torch
        if out is None:
            out = torch.empty((self.n, self.n), dtype=torch.float64, device=self.A.device,
                              pin_memory=not self.A.is_cuda)
        _check_matrix(out, self.n, "finalize: out", self.A, host_ok=True)
        ctx, self.ctx = self.ctx, None
        ipr_finalize(ctx, out, out.stride(0))
        return out

    def close(self):
        if self.ctx is not None:
            ctx, self.ctx = self.ctx, None
            ipr_finalize(ctx)

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def solve(A, p: int, phases, final_tol: float = 1e-12, max_iters: int = 1000, stream=None,
          form="literal", cert="fp64"):
    """Run a full solve; returns (C_best, outcome name, trace)."""
    s = Solver(A, p, phases, final_tol, stream, form=form, cert=cert)
    s.iterate(max_iters)
    tr = s.trace()
    out = OUTCOME_NAMES[s.outcome]
    return s.finalize(), out, tr
