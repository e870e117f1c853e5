"""Pins of the oracle controller (reading R-5 of DESIGN.md; "the necessity of
increased precision can be detected at runtime").  Decisions below were worked out by hand from
the rule text, for n = 4 (rho_hat = rho / 2)."""
import math

import oracle

C, CV, IL, DV, NF, SW = (oracle.CONTINUE, oracle.CONVERGED, oracle.ITER_LIMIT, oracle.DIVERGED,
                         oracle.NONFINITE, oracle.SWITCH)


def run(phases, seq, final_tol=1e-12):
    ctl = oracle.Controller(4, len(phases), final_tol)
    out = []
    for rho in seq:
        d = ctl.decide(phases[ctl.c.phase], rho)
        out.append((d, ctl.best_is_new))
        if d == SW:
            ctl.next_phase()
    return out


LOW = oracle.phase(oracle.BF16, switch_tol=1e-3, plateau_ratio=0.7, plateau_arm=0.5, max_iters=10)
HIGH = oracle.phase(oracle.FP64)


def test_armed_plateau_then_convergence():
    # 8.0: rho_hat 4 (unarmed) -> continue; 7.9 continue; 0.9: armed (0.45<0.5) but 0.9 < 0.7*7.9;
    # 0.8: armed and 0.8 > 0.63 -> switch; FP64: 0.5 continue, 1e-13 <= 1e-12 converged.
    got = run([LOW, HIGH], [8.0, 7.9, 0.9, 0.8, 0.5, 1e-13])
    assert [d for d, _ in got] == [C, C, C, SW, C, CV]
    assert [b for _, b in got] == [True, True, True, True, True, True]


def test_unarmed_plateau_does_not_fire():
    # rho_hat stays >= 0.5: growth 7.9 -> 7.95 would trip an un-armed rule (SURVEY Table A4).
    got = run([LOW, HIGH], [8.0, 7.9, 7.95, 7.0])
    assert [d for d, _ in got] == [C, C, C, C]
    assert [b for _, b in got] == [True, True, False, True]


def test_switch_tol():
    got = run([LOW, HIGH], [8.0, 1e-3])
    assert [d for d, _ in got] == [C, SW]


def test_divergence_last_phase_and_nonlast():
    # min rho_hat 0.1 (rho 0.2); 3.0 -> rho_hat 1.5 > 10*0.1 and > 1 -> diverged / switch
    assert [d for d, _ in run([HIGH], [1.0, 0.2, 3.0])] == [C, C, DV]
    assert [d for d, _ in run([LOW, HIGH], [1.0, 0.2, 3.0])][:3] == [C, C, SW]
    # 1.9 -> rho_hat 0.95 not > 1: no divergence
    assert [d for d, _ in run([HIGH], [1.0, 0.2, 1.9])] == [C, C, C]


def test_nonfinite():
    assert [d for d, _ in run([LOW, HIGH], [8.0, math.nan])] == [C, SW]
    assert [d for d, _ in run([HIGH], [8.0, math.inf])] == [C, NF]


def test_phase_cap():
    cap = oracle.phase(oracle.FP64, max_iters=2)
    assert [d for d, _ in run([cap], [5.0, 4.0])] == [C, IL]
    low2 = oracle.phase(oracle.BF16, max_iters=2)
    assert [d for d, _ in run([low2, HIGH], [5.0, 4.0, 3.0])] == [C, SW, C]


def test_final_tol_only_in_last_phase():
    # a low phase never "converges"; 1e-13 <= switch_tol -> switch
    assert [d for d, _ in run([LOW, HIGH], [1e-13])] == [SW]
    nothing = oracle.phase(oracle.BF16)
    assert [d for d, _ in run([nothing, HIGH], [1e-13, 1e-13])] == [C, C]
