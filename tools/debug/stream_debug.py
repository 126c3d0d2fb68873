"""Locate wrong outputs of hvp_stream_kernel: tile / lane pattern for several m."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_2410_22575_b200 as chf, oracle, synth
dev = torch.device("cuda")
for n in (2, 4, 8):
    for m in (256 * 300, 256 * 600 + 17, 600011):
        P, V = synth.points(30, n, m), synth.vectors(30, n, m)
        ref, sabs = oracle.hvp_batch("rosenbrock", P, V, 1, None)
        for C in (1, n):
            got = chf.hvp_batch("rosenbrock", torch.from_numpy(P).to(dev), torch.from_numpy(V).to(dev), C).cpu().numpy()
            err = oracle.componentwise_error(got, ref, sabs).max(axis=1)
            bad = np.nonzero(err > 1e-10)[0]
            msg = f"n={n} m={m} C={C}: bad {bad.size}"
            if bad.size:
                tiles = np.unique(bad // 256)
                msg += f" tiles {tiles[:10]} (#{tiles.size}) lanes {np.unique(bad % 256)[:8]} first {bad[:5]}"
                # is a bad row equal to the reference of another point?
                b = bad[0]
                hit = np.nonzero(np.all(np.abs(ref - got[b]) < 1e-9 * (1 + np.abs(ref)), axis=1))[0]
                msg += f" got[b]==ref of {hit[:5]}"
            print(msg, flush=True)
