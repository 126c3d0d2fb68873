"""One launch of one (func, n, C, algo) for ncu --set full captures (after 2 warm-up launches).

    ncu --set full --import-source on -k regex:hvp_ -c 1 -s 2 python tools/prof_one.py rosenbrock 16 16 [hvp] [m]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2410_22575_b200 as chf  # noqa: E402
import synth  # noqa: E402

func, n, C = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
algo = sys.argv[4] if len(sys.argv) > 4 else "hvp"
m = int(sys.argv[5]) if len(sys.argv) > 5 else 1 << 20
dev = torch.device("cuda", 0)
p = torch.from_numpy(synth.points(0, n, m)).to(dev)
v = torch.from_numpy(synth.vectors(0, n, m)).to(dev)
pr = torch.from_numpy(synth.fp_params_flat(0, n)).to(dev) if func == "fletcher_powell" else None
fn = {"hvp": chf.hvp_batch, "sym_hvp": chf.sym_hvp_batch, "hvp_hoisted": chf.hvp_batch_hoisted,
      "hvp_seedsparse": chf.hvp_batch_seedsparse}
for _ in range(3):
    if algo in fn:
        fn[algo](func, p, v, C, pr)
    else:
        getattr(chf, algo + "_batch")(func, p, C, pr)
torch.cuda.synchronize()
print("kernel path:", chf.path(func, n, C, algo if algo in chf.ALGOS else "hvp"))
