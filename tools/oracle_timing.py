"""The oracle (test infrastructure, oracle/) timed on one full solve of the headline schedule at several
orders (kappa = 2 twins, seed 5): the measured CPU baseline behind bench.py's cpu_baseline scaling.
python tools/oracle_timing.py [n ...]  -> one JSON line per order."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import bench
    import oracle
    import synth
    ns = [int(x) for x in sys.argv[1:]] or [1024, 2048, 4096]
    for n in ns:
        A = synth.spd(n, 2.0, 5)
        oform, ph = bench.oracle_schedule(bench.DEFAULT_SCHEDULE, n)
        t0 = time.perf_counter()
        r = oracle.solve(A, 2, ph, 1e-12, 300, form=oform)
        t = time.perf_counter() - t0
        cert = [x["rho_cert"] for x in r.records if x["rho_cert"] == x["rho_cert"]]
        print(json.dumps({"n": n, "schedule": bench.DEFAULT_SCHEDULE, "outcome": oracle.OUTCOME_NAMES[r.outcome],
                          "iters_per_phase": [sum(1 for x in r.records if x["phase"] == i) for i in range(len(ph))],
                          "gemms": bench.oracle_gemms(r.records, 2), "rho_cert": cert[-1] if cert else None,
                          "seconds": t, "threads": len(os.sched_getaffinity(0))}), flush=True)


if __name__ == "__main__":
    main()
