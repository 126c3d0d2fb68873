import sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_2410_22575_b200 as chf, synth
for n, m in ((2, 100), (8, 70), (32, 50)):
    P = synth.points(21, n, m); params = synth.fp_params_flat(0, n)
    p, pr = torch.from_numpy(P).cuda(), torch.from_numpy(params).cuda()
    a = chf.hessian_batch("fletcher_powell", p, n, pr).cpu().numpy()
    b = chf.hessian_batch_seedsparse("fletcher_powell", p, n, pr).cpu().numpy()
    d = a != b
    rel = np.abs(a - b) / np.maximum(np.abs(a), 1e-300)
    print(n, "mismatch", d.sum(), "of", d.size, "max rel", rel.max())
    ii, jj = np.nonzero(d.any(axis=0))
    print("  positions (i,j):", list(zip(ii.tolist(), jj.tolist()))[:20])
    diag = np.eye(n, dtype=bool)
    print("  diag mismatches", d[:, diag].sum(), "offdiag", d[:, ~diag].sum(), "row0", d[:, 0, :].sum(), "col0", d[:, :, 0].sum())
    vh = chf.hvp_batch_seedsparse("fletcher_powell", p, torch.from_numpy(synth.vectors(21, n, m)).cuda(), n, pr).cpu().numpy()
    va = chf.hvp_batch("fletcher_powell", p, torch.from_numpy(synth.vectors(21, n, m)).cuda(), n, pr).cpu().numpy()
    print("  hvp mismatch", (vh != va).sum(), "max rel", (np.abs(vh - va) / np.abs(va)).max())
