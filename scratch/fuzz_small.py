"""A short block of every fuzz kind (for compute-sanitizer runs)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_2501_12369_b200 as darbs
from oracle import cpu
import fuzz_cases as F
port, ctx = cpu.load("port"), darbs.Context(0)
n = int(sys.argv[1])
print("raster", sum(F.trial(ctx, port, s) for s in range(n)), "chain", sum(F.chain_trial(ctx, port, darbs, s) for s in range(n)),
      "bins", sum(F.bins_trial(ctx, port, s) for s in range(max(1, n // 4))), "loss", sum(F.loss_trial(ctx, port, s) for s in range(n)), "of", n)
