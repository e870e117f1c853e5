import sys; sys.path.insert(0, '/root/repo')
import torch, numpy as np, bench, synth, paper_1703_02283_b200 as ipr
n = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
A, _ = synth.spd_torch(n, 2.0, 5, device="cuda")
form, ph = bench.schedule(bench.DEFAULT_SCHEDULE, n)
outs = []
for r in range(3):
    s = ipr.Solver(A, 2, ph, 1e-12, form=form, cert="crt")
    s.iterate(1)
    npad = (n + 255) // 256 * 256
    z = ipr.ipr_test_peek(s.ctx, ipr.IPR_PEEK_Z1, npad).cpu().numpy()
    rh = ipr.ipr_test_peek(s.ctx, ipr.IPR_PEEK_RHAT, npad).cpu().numpy()
    outs.append((z, rh, s.trace()[0]["rho"]))
    s.close()
for r in (1, 2):
    dz = outs[r][0] != outs[0][0]
    dr = outs[r][1] != outs[0][1]
    print("rep", r, "Z1 diffs", int(dz.sum()), "R diffs", int(dr.sum()), "rho", outs[r][2], outs[0][2])
    if dz.any():
        ii, jj = np.nonzero(dz)
        print("  Z1 diff (buffer [k][j]) rows", ii[:10], "cols", jj[:10], "upper(k<j)", int((ii < jj).sum()), "lower", int((ii > jj).sum()), "diag", int((ii == jj).sum()))
        print("  tiles", sorted(set(zip((ii // 256).tolist(), (jj // 256).tolist())))[:20])
