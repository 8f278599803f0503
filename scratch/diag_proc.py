import sys, numpy as np
sys.path.insert(0, "tests")
from conftest import scene_f32
import conftest
from oracle import cpu
import paper_2501_12369_b200 as d
port = cpu.load("port")
ctx = d.Context(0)
name = sys.argv[1] if len(sys.argv) > 1 else "raised-cosine"
n, w, h, seed = 3000, 77, 45, 11
k = port.preset(name)
s = port.random_scene(k, n, w, h, seed)
ref = port.forward(k, s, w, h, (0.1, 0.2, 0.3), threads=0)
out = ctx.forward(d.kernel_preset(name), **scene_f32(s), width=w, height=h, background=(0.1, 0.2, 0.3))
wc = ctx.work_counters()
bad = np.argwhere(out["processed"] != ref["processed"])
print("bad", len(bad), "wc", wc)
for y, x in bad[:10]:
    print(y, x, "proc", out["processed"][y, x], ref["processed"][y, x], "contrib", out["contributors"][y, x],
          ref["contributors"][y, x], "T", out["t_final"][y, x], ref["t_final"][y, x])
