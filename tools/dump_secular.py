"""Dev helper: dump deflated secular problems (K, rho, poles, weights, per-root
iteration counts) of the event kernel at the cfg-5 steady state, 8 per reset
(DAMF_PROF build): DAMF_GPU_LIB=.../libdamf_gpu_prof.so python tools/dump_secular.py [rounds]"""
import ctypes as C
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
from paper_2306_08967_b200 import engine as ge
from paper_2306_08967_b200 import workloads as W
from test_gpu_configs import cfg5_like

rounds = int(sys.argv[1]) if len(sys.argv) > 1 else 40
e, su, sv = cfg5_like(20, 128, 200 + 2 * rounds, seed=4)
e.apply(W.EventList.edges(1, su[:200], sv[:200]))
L = ge.lib()
L.damf_gpu_debug_dump.argtypes = [C.c_void_p, C.c_void_p, C.c_int64]
out = []
for r in range(rounds):
    L.damf_gpu_debug_dump(e.h, None, -1)
    e.apply(W.EventList.edges(1, su[200 + 2 * r:202 + 2 * r], sv[200 + 2 * r:202 + 2 * r]))
    buf = np.zeros(8 + 8 * 800)
    L.damf_gpu_debug_dump(e.h, buf.ctypes.data, len(buf))
    out.append(buf[8:].reshape(8, 800).copy())
out = np.concatenate(out)
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
np.save(os.path.join(root, "gpurun_out", "secular_problems.npy"), out)
its = np.array([o[530:530 + int(o[0])].max() for o in out if o[0] > 0])
print("problems", len(its), "max its per problem: mean %.2f p50 %d p90 %d max %d" %
      (its.mean(), np.median(its), np.percentile(its, 90), its.max()))
