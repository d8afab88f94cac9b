"""Diagnostic: device adapt_full_data over several seeds vs the stored reference fit."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "tests"), os.path.join(ROOT, "tests", "golden")):
    sys.path.insert(0, p)
import numpy as np
from parity_util import Case
import make_golden
from paper_2310_07002_b200 import pcv
for name in sys.argv[1:]:
    c = Case(name); akw = make_golden.CONFIGS[name][1]
    cfg = pcv.AdaptConfig(chains=akw["chains"], warmup=akw["warmup"], draws=akw["draws"])
    rb = c.z["bank0"]
    with pcv.Context(0) as ctx:
        for s in (1, 2, 3, 4):
            f = ctx.adapt_full_data(c.models[0], cfg, seed=s, model_id=0)
            sd = np.sqrt(0.5 * (f.draws.var(0) + rb.var(0)))
            z = np.abs(f.draws.mean(0) - rb.mean(0)) / sd
            print(name, s, "step %.4f" % f.kparams.step_size, "ref %.4f" % float(c.z["step0"]),
                  "accept %.3f" % f.mean_accept, "mass ratio med %.3f" % np.median(f.kparams.inv_mass_diag / c.z["inv_mass0"]),
                  "|dmean|/sd med %.3f max %.3f" % (np.median(z), z.max()), "ms %.1f" % f.device_ms, flush=True)
