import sys, numpy as np
sys.path.insert(0, '/root/repo')
from paper_1902_07554_b200 import gpu, host
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
inst = host.make_instance(3, n=n, k=64)
ctx = gpu.Context(0)
res = gpu.assign_points(inst.points, inst.sample_ids, inst.sample_labels, 64, ctx=ctx)
print("ok", n, res.labels[:5])
