"""Replay a sequence of chain seeds in ONE context (state carried between trials), repeated."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_2501_12369_b200 as darbs
from oracle import cpu
import fuzz_cases as F
port, ctx = cpu.load("port"), darbs.Context(0)
seeds = [int(a) for a in sys.argv[1:]]
for rep in range(3):
    print("rep", rep, [(s, F.chain_trial(ctx, port, darbs, s)) for s in seeds], flush=True)
