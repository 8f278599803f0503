import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_2501_12369_b200 as darbs
from oracle import cpu
import fuzz_cases as F
port, ctx = cpu.load("port"), darbs.Context(0)
kind = sys.argv[1]
for s in sys.argv[2:]:
    s = int(s)
    ok = {"raster": lambda: F.trial(ctx, port, s), "chain": lambda: F.chain_trial(ctx, port, darbs, s), "loss": lambda: F.loss_trial(ctx, port, s)}[kind]()
    print(kind, s, ok)
