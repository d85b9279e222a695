"""ncu target: warm + profiled prepare_device launches for one config (env CFG=cfg3|cfg4)."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2203_07747_b200 import _lib, make_mlp, synth_quad_nodes
from paper_2203_07747_b200.errors import raise_for_status
cfg = os.environ.get("CFG", "cfg3")
sizes, seed, k = ([17] + [512] * 12 + [6], 12512, 20) if cfg == "cfg3" else ([17] + [256] * 5 + [6], 5256, 81920)
m = make_mlp(sizes, "silu", "full", seed)
eng = m.engine(latency_mode=1 if cfg == "cfg3" else 0)
eng._ensure(k, 1)
z = torch.from_numpy(synth_quad_nodes(3, k)).cuda()
f = torch.empty((k, 6), dtype=torch.float64, device="cuda")
j = torch.empty((k, 6, 17), dtype=torch.float64, device="cuda")
L = _lib.lib()
for _ in range(int(os.environ.get("REPS", 3))):
    raise_for_status(L.rtn_prepare_device(eng.ctx_ptr, z.data_ptr(), k, 1, f.data_ptr(), j.data_ptr(), None))
torch.cuda.synchronize()
print("done", cfg)
