import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle
import paper_1502_00512_b200 as dl
V, H = int(sys.argv[1]), int(sys.argv[2])
orc = oracle.Orc()
params = orc.init_uniform(V, H, 4)
ids = orc.random_stream(9, V, 40000)
m = dl.GpuRnn(V, H, 0, "bf16")
m.set_params(*params)
m.set_opt(None, None, None, 0.9995, 1e-6)
m.trainer_init(ids, 4, 64, 8, 1.0)
m.set_profiling(True)
print(m.trainer_run(0, 1, 0.01))
