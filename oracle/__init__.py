"""TEST INFRASTRUCTURE ONLY -- ctypes binding of the plain-C FP64 oracle (oracle/ipr_oracle.c).

Only tests/, ``__graft_entry__.smoke()`` and bench.py's ``cpu_baseline`` / ``--impl reference``
legs may import this module.  The CUDA product path (``paper_1703_02283_b200``) never imports,
links or executes anything under ``oracle/``; the two share no code.

Every function cites the PAPER.md passage it follows (see ipr_oracle.h / ipr_oracle.c).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "ipr_oracle.c")
_LIB = os.path.join(_HERE, "libipr_oracle.so")

FP64, TF32, BF16, FP16, FP8, INT8, FP64_OZ, FP64_CRT = 0, 1, 2, 3, 4, 5, 6, 7
MANT_ADAPTIVE = -2   # FP64_OZ / FP64_CRT phases: digits / stored bits chosen per iteration (reading R-26)
RNE, RTZ = 0, 1
CONTINUE, CONVERGED, ITER_LIMIT, DIVERGED, NONFINITE, SWITCH = 0, 1, 2, 3, 4, 5
OUTCOME_NAMES = {0: "running", 1: "converged", 2: "iter_limit", 3: "diverged", 4: "nonfinite",
                 5: "switch"}


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (-ffp-contract=off: no FMA contraction)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < max(
            os.path.getmtime(_SRC), os.path.getmtime(os.path.join(_HERE, "ipr_oracle.h"))):
        cmd = ["gcc", "-O3", "-fopenmp", "-ffp-contract=off", "-fno-fast-math", "-fPIC",
               "-shared", "-std=c11", "-Wall", "-o", _LIB + ".tmp", _SRC, "-lm"]
        subprocess.check_call(cmd)
        os.replace(_LIB + ".tmp", _LIB)
    return _LIB


class Phase(C.Structure):
    _fields_ = [("prec", C.c_int), ("mant_bits", C.c_int), ("round", C.c_int),
                ("switch_tol", C.c_double), ("plateau_ratio", C.c_double),
                ("plateau_arm", C.c_double), ("max_iters", C.c_int), ("corr_prec", C.c_int)]


class Record(C.Structure):
    _fields_ = [("k", C.c_int), ("phase", C.c_int), ("prec", C.c_int), ("mant_bits", C.c_int),
                ("decision", C.c_int), ("rho", C.c_double), ("rho_hat", C.c_double),
                ("delta", C.c_double), ("gamma", C.c_double), ("rho_cert", C.c_double)]


class Ctrl(C.Structure):
    _fields_ = [("phase", C.c_int), ("nphases", C.c_int), ("it_in_phase", C.c_int),
                ("n", C.c_int64), ("rho_prev", C.c_double), ("rho_best", C.c_double),
                ("rhohat_min", C.c_double), ("final_tol", C.c_double),
                ("best_is_new", C.c_int)]


_lib = None
_dp = C.POINTER(C.c_double)


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        L = _lib
        L.orc_qm.restype = C.c_double
        L.orc_qm.argtypes = [C.c_double, C.c_int, C.c_int, C.c_int]
        L.orc_qm_array.argtypes = [C.c_int64, _dp, _dp, C.c_int, C.c_int, C.c_int]
        L.orc_norms.argtypes = [C.c_int64, _dp, _dp]
        L.orc_is_symmetric.argtypes = [C.c_int64, _dp]
        L.orc_gemm.argtypes = [C.c_int64, _dp, _dp, _dp]
        L.orc_matvec.argtypes = [C.c_int64, _dp, _dp, _dp]
        L.orc_gemm_rows.argtypes = [C.c_int64, C.c_int64, C.c_int64, _dp, _dp, _dp]
        L.orc_gemm_cols.argtypes = [C.c_int64, C.c_int64, C.c_int64, _dp, _dp, _dp]
        L.orc_c0.argtypes = [C.c_int64, _dp, C.c_double, C.POINTER(Phase), _dp]
        L.orc_step.restype = C.c_double
        L.orc_step.argtypes = [C.c_int64, C.c_int, _dp, _dp, C.POINTER(Phase), _dp, _dp]
        L.orc_solve.argtypes = [C.c_int64, C.c_int, _dp, C.POINTER(Phase), C.c_int, C.c_double,
                                C.c_int, C.POINTER(Record), C.c_int, C.POINTER(C.c_int), _dp,
                                _dp, C.c_int, C.c_double, _dp]
        L.orc_solve_form.argtypes = [C.c_int64, C.c_int, C.c_int, _dp, C.POINTER(Phase), C.c_int,
                                     C.c_double, C.c_int, C.POINTER(Record), C.c_int,
                                     C.POINTER(C.c_int), _dp, _dp, C.c_int, C.c_double, _dp]
        L.orc_step_sym.restype = C.c_double
        L.orc_step_sym.argtypes = [C.c_int64, C.c_int, _dp, _dp, C.POINTER(Phase), _dp, _dp]
        L.orc_step_sym_form.restype = C.c_double
        L.orc_step_sym_form.argtypes = [C.c_int64, C.c_int, C.c_int, _dp, _dp, C.POINTER(Phase), _dp, _dp]
        L.orc_step_ns.restype = C.c_double
        L.orc_step_ns.argtypes = [C.c_int64, _dp, _dp, C.POINTER(Phase), _dp, _dp]
        L.orc_jacobi.argtypes = [C.c_int64, _dp, _dp, _dp]
        L.orc_set_predict_cert.argtypes = [C.c_int]
        L.orc_set_cert_mode.argtypes = [C.c_int]
        L.orc_cert_grid.argtypes = [C.c_int64, C.c_int, _dp, _dp]
        L.orc_resid_dd.restype = C.c_double
        L.orc_resid_dd.argtypes = [C.c_int64, C.c_int, _dp, _dp]
        L.orc_resid_rows_dd.argtypes = [C.c_int64, C.c_int, _dp, _dp, C.c_int64, C.POINTER(C.c_int64), _dp]
        L.orc_inv_proot_eig.argtypes = [C.c_int64, _dp, _dp, C.c_int, _dp]
        L.orc_spectral.argtypes = [C.c_int64, _dp, C.c_int, C.c_double, C.c_int, _dp]
        L.orc_fp16_sigma.argtypes = [C.c_double]
        L.orc_sigma.argtypes = [C.c_int, C.c_double]
        L.orc_oz_digits.argtypes = [C.c_double, C.c_int64]
        L.orc_oz_adaptive_m.argtypes = [C.c_int]
        L.orc_digits_for_m.argtypes = [C.c_int]
        L.orc_crt_bits.argtypes = [C.c_int, C.c_int64]
        L.orc_gemm_crt.argtypes = [C.c_int64, C.c_int, _dp, _dp, _dp]
        L.orc_gemm_crt_pairs.argtypes = [C.c_int64, C.c_int, _dp, _dp, C.c_int64, C.POINTER(C.c_int64),
                                         C.POINTER(C.c_int64), _dp]
        L.orc_q_int8.restype = C.c_double
        L.orc_q_int8.argtypes = [C.c_double]
        L.orc_ctrl_init.argtypes = [C.POINTER(Ctrl), C.c_int64, C.c_int, C.c_double]
        L.orc_ctrl_decide.argtypes = [C.POINTER(Ctrl), C.POINTER(Phase), C.c_double]
        L.orc_ctrl_enter_next_phase.argtypes = [C.POINTER(Ctrl)]
        L.orc_prec_format.argtypes = [C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int)]
        L.orc_container_E.argtypes = [C.c_int]
        L.orc_native_m.argtypes = [C.c_int]
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(_dp)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def phase(prec=FP64, mant_bits=-1, round=RNE, switch_tol=0.0, plateau_ratio=0.0,
          plateau_arm=0.5, max_iters=0, corr_prec=-1) -> Phase:
    """corr_prec: operand format of the correction GEMM of FORM_SYMMETRIC (-1 = prec)."""
    return Phase(prec, mant_bits, round, switch_tol, plateau_ratio, plateau_arm, max_iters,
                 corr_prec)


def qm(x, E: int, m: int, rtz: bool = False) -> np.ndarray:
    """q_m of PAPER.md:191-194 (custom exponent/mantissa widths), elementwise."""
    x = _f64(x)
    y = np.empty_like(x)
    lib().orc_qm_array(x.size, _p(x), _p(y), E, m, int(rtz))
    return y


def prec_format(prec: int):
    E, M = C.c_int(), C.c_int()
    lib().orc_prec_format(prec, C.byref(E), C.byref(M))
    return E.value, M.value


def container_E(prec: int) -> int:
    return lib().orc_container_E(prec)


def native_m(prec: int) -> int:
    return lib().orc_native_m(prec)


def fp16_sigma(maxabs: float) -> int:
    return lib().orc_fp16_sigma(maxabs)


def sigma(prec: int, maxabs: float) -> int:
    """Scale exponent of the scaled operand formats (FP16 / FP8 / INT8), 0 otherwise."""
    return lib().orc_sigma(prec, maxabs)


def oz_digits(rho_hat_target: float, n: int) -> int:
    return lib().orc_oz_digits(rho_hat_target, n)


def oz_adaptive_m(S: int) -> int:
    return lib().orc_oz_adaptive_m(S)


def digits_for_m(m: int) -> int:
    """Digits S of a fixed-m FP64_OZ / FP64_CRT phase (reading R-23)."""
    return lib().orc_digits_for_m(m)


def crt_bits(S: int, n: int) -> int:
    """Bits b of an FP64_CRT product with S Ozaki-equivalent digits at order n (reading R-28)."""
    return lib().orc_crt_bits(S, n)


def gemm_crt(X, Y, b: int) -> np.ndarray:
    """Z = X (x)_b Y: rows of X / columns of Y quantised to b-bit integers relative to their maximum,
    the integer product exact, one rounding (reading R-28; the definition the GPU's CRT GEMM emulates)."""
    X, Y = _f64(X), _f64(Y)
    Z = np.empty_like(X)
    lib().orc_gemm_crt(X.shape[0], int(b), _p(X), _p(Y), _p(Z))
    return Z


def gemm_crt_pairs(X, Y, b: int, I, J) -> np.ndarray:
    """Elements (I[q], J[q]) of gemm_crt(X, Y, b), exponents from the full rows / columns."""
    X, Y = _f64(X), _f64(Y)
    I = np.ascontiguousarray(I, dtype=np.int64)
    J = np.ascontiguousarray(J, dtype=np.int64)
    Z = np.empty(I.shape[0])
    lib().orc_gemm_crt_pairs(X.shape[0], int(b), _p(X), _p(Y), I.shape[0],
                             I.ctypes.data_as(C.POINTER(C.c_int64)), J.ctypes.data_as(C.POINTER(C.c_int64)), _p(Z))
    return Z


def q_int8(x: float) -> float:
    """INT8 fixed-point quantiser: nearest-even integer saturated to [-127, 127]."""
    return lib().orc_q_int8(x)


def norms(A):
    """(||A||_1, ||A||_inf, max diag) of Eq. (3)."""
    A = _f64(A)
    out = np.empty(3)
    lib().orc_norms(A.shape[0], _p(A), _p(out))
    return float(out[0]), float(out[1]), float(out[2])


def is_symmetric(A) -> bool:
    A = _f64(A)
    return bool(lib().orc_is_symmetric(A.shape[0], _p(A)))


def gemm(X, Y) -> np.ndarray:
    X, Y = _f64(X), _f64(Y)
    Z = np.empty_like(X)
    lib().orc_gemm(X.shape[0], _p(X), _p(Y), _p(Z))
    return Z


def gemm_rows(X, Y, Z, r0: int, r1: int) -> None:
    """Rows [r0, r1) of Z = X Y in place (bounded timing sample; same loops as gemm)."""
    lib().orc_gemm_rows(X.shape[0], r0, r1, _p(X), _p(Y), _p(Z))


def gemm_cols(X, Y, Z, c0: int, c1: int) -> None:
    """Columns [c0, c1) of Z = X Y in place (same per-element k order as gemm)."""
    lib().orc_gemm_cols(X.shape[0], c0, c1, _p(X), _p(Y), _p(Z))


def matvec(X, v) -> np.ndarray:
    X, v = _f64(X), _f64(v)
    y = np.empty(X.shape[0])
    lib().orc_matvec(X.shape[0], _p(X), _p(v), _p(y))
    return y


def c0(A, s: float, ph0: Phase) -> np.ndarray:
    A = _f64(A)
    out = np.empty_like(A)
    lib().orc_c0(A.shape[0], _p(A), s, C.byref(ph0), _p(out))
    return out


def step(A, Ck, p: int, ph: Phase, want_next: bool = True):
    """One Eq. (1) iteration from C_k: returns (rho(C_k), C_{k+1}, delta)."""
    A, Ck = _f64(A), _f64(Ck)
    nxt = np.empty_like(Ck) if want_next else None
    d = C.c_double(np.nan)
    rho = lib().orc_step(A.shape[0], p, _p(A), _p(Ck), C.byref(ph),
                         _p(nxt) if want_next else None, C.byref(d))
    return rho, nxt, d.value


class SolveResult:
    def __init__(self, outcome, records, C_best, C_hist, s):
        self.outcome = outcome
        self.records = records
        self.C_best = C_best
        self.C_hist = C_hist
        self.s = s

    @property
    def rho(self):
        return np.array([r["rho"] for r in self.records])


def step_ns(A, Xk, ph: Phase, want_next: bool = True):
    """One Newton-Schulz step X (2I - A X) (NEXT-1): returns (rho(X_k), X_{k+1}, delta)."""
    A, Xk = _f64(A), _f64(Xk)
    nxt = np.empty_like(Xk) if want_next else None
    d = C.c_double(np.nan)
    rho = lib().orc_step_ns(A.shape[0], _p(A), _p(Xk), C.byref(ph),
                            _p(nxt) if want_next else None, C.byref(d))
    return rho, nxt, d.value


def step_sym(A, Ck, p: int, ph: Phase, want_next: bool = True, tri: bool = False):
    """One symmetrised-correction step (NEXT-2, p >= 2): C + (W + W^T)/(2p), W = qc(C) qc(I - Z_p),
    Z_p = C^{p-1} A C.  tri: the symmetric-tri form (p = 2; R-36 below the FP64 range); tri = 2: a chain
    of FORM_SYMMETRIC_TRIZ whose Z_1 is taken from its upper triangle too (R-37).
    Returns (rho_s(C_k) = ||I - Z_p||_F, C_{k+1}, delta)."""
    A, Ck = _f64(A), _f64(Ck)
    nxt = np.empty_like(Ck) if want_next else None
    d = C.c_double(np.nan)
    rho = lib().orc_step_sym_form(A.shape[0], p, int(tri), _p(A), _p(Ck), C.byref(ph),
                                  _p(nxt) if want_next else None, C.byref(d))
    return rho, nxt, d.value


FORM_LITERAL, FORM_NEWTON_SCHULZ, FORM_SYMMETRIC, FORM_SYMMETRIC_TRI, FORM_COUPLED = 0, 1, 2, 3, 4
FORM_SYMMETRIC_TRIZ = 5   # reading R-37: the tri form + Z_1 from its upper triangle in fast FP64_CRT phases


def solve(A, p: int, phases, final_tol: float = 1e-12, max_total: int = 200,
          hist: int = 0, gamma_normA2: float = 0.0, form: int = FORM_LITERAL,
          predict_cert: bool = True, cert: str = "fp64") -> SolveResult:
    """Full controller-driven solve (init + iterations), reading R-5 of DESIGN.md.
    form = FORM_LITERAL (Eq. 1 as printed), FORM_NEWTON_SCHULZ (p = 1, X(2I - AX)) or
    FORM_SYMMETRIC (p >= 2, C + (W + W^T)/(2p); convergence certified on ||I - C^p A||_F).
    predict_cert: reading R-33 (certificate-first iterates in the symmetric forms' last phase; the
    GPU's IPR_CERT_FP64) -- False mirrors IPR_CERT_FP64_CHAIN.
    cert: "fp64" (R-30: the FP64 literal chain) or "crt" (R-35: the candidate's grid rounding
    cert_grid(C, 62) certified by its double-double residual; that matrix is the answer)."""
    A = _f64(A)
    lib().orc_set_predict_cert(1 if predict_cert else 0)
    lib().orc_set_cert_mode({"fp64": 0, "dmma": 0, "crt": 1}[cert])
    n = A.shape[0]
    arr = (Phase * len(phases))(*phases)
    recs = (Record * max_total)()
    nrec = C.c_int(0)
    best = np.empty_like(A)
    H = np.empty((hist, n, n)) if hist > 0 else None
    s = C.c_double(0)
    out = lib().orc_solve_form(n, p, form, _p(A), arr, len(phases), final_tol, max_total, recs,
                               max_total, C.byref(nrec), _p(best),
                               _p(H) if H is not None else None, hist, gamma_normA2, C.byref(s))
    if out < 0:
        raise ValueError({-1: "invalid argument", -2: "A is not exactly symmetric"}[out])
    records = [dict(k=r.k, phase=r.phase, prec=r.prec, mant_bits=r.mant_bits,
                    decision=r.decision, rho=r.rho, rho_hat=r.rho_hat, delta=r.delta,
                    gamma=r.gamma, rho_cert=r.rho_cert) for r in recs[:min(nrec.value, max_total)]]
    return SolveResult(out, records, best, H, s.value)


def cert_grid(C_, b: int = 62) -> np.ndarray:
    """Reading R-35: C rounded to the coarser of its row's and column's b-bit grids (ipr_oracle.h)."""
    X = _f64(C_)
    out = np.empty_like(X)
    lib().orc_cert_grid(X.shape[0], b, _p(X), _p(out))
    return out


def resid_dd(A, X, p: int) -> float:
    """||I - X^p A||_F in double-double arithmetic (the residual of the FP64 matrices X, A to ~1e-30)."""
    A, X = _f64(A), _f64(X)
    return lib().orc_resid_dd(A.shape[0], p, _p(A), _p(X))


def resid_rows_dd(A, X, p: int, rows) -> np.ndarray:
    """Squared 2-norms of the given rows of I - X^p A, in double-double arithmetic (sampled rows)."""
    A, X = _f64(A), _f64(X)
    r = np.ascontiguousarray(rows, dtype=np.int64)
    out = np.empty(len(r))
    lib().orc_resid_rows_dd(A.shape[0], p, _p(A), _p(X), len(r), r.ctypes.data_as(C.POINTER(C.c_int64)), _p(out))
    return out


def jacobi(A):
    """Cyclic Jacobi eigen-decomposition (SPEC.md oracle module): (lambda asc, V)."""
    A = _f64(A)
    n = A.shape[0]
    lam, V = np.empty(n), np.empty_like(A)
    lib().orc_jacobi(n, _p(A), _p(lam), _p(V))
    return lam, V


def inv_proot_eig(lam, V, p: int) -> np.ndarray:
    lam, V = _f64(lam), _f64(V)
    X = np.empty_like(V)
    lib().orc_inv_proot_eig(V.shape[0], _p(lam), _p(V), p, _p(X))
    return X


def spectral(lam, p: int, s: float, kmax: int) -> np.ndarray:
    lam = _f64(lam)
    out = np.empty(kmax)
    lib().orc_spectral(lam.size, _p(lam), p, s, kmax, _p(out))
    return out


class Controller:
    """Pure controller state machine of reading R-5 (for direct tests)."""

    def __init__(self, n: int, nphases: int, final_tol: float):
        self.c = Ctrl()
        lib().orc_ctrl_init(C.byref(self.c), n, nphases, final_tol)

    def decide(self, ph: Phase, rho: float) -> int:
        return lib().orc_ctrl_decide(C.byref(self.c), C.byref(ph), rho)

    def next_phase(self):
        lib().orc_ctrl_enter_next_phase(C.byref(self.c))

    @property
    def best_is_new(self) -> bool:
        return bool(self.c.best_is_new)
