import sys, os; sys.path.insert(0, '.')
import numpy as np, torch, ctypes
import paper_2603_28770_b200 as z
from paper_2603_28770_b200 import engine, _capi
from paper_2603_28770_b200.linesearch import LineSearchParams
dev = torch.device("cuda", 0)
d, n = 50, 8
x0 = torch.rand((d, n), dtype=torch.float64, device=dev) * 4 - 2
out = engine.BfgsBuffers.allocate(d, n, dev)
print("launch", flush=True)
L = _capi.lib()
ws = torch.zeros(1024, dtype=torch.uint8, device=dev)
P = engine.bfgs_params(1e-6, 60, LineSearchParams())
rc = L.zeus_bfgs(2, d, n, x0.data_ptr(), n, P, 0, None, None, out.c_struct(n), ws.data_ptr(), torch.cuda.current_stream().cuda_stream)
print("rc", rc, L.zeus_last_error(), flush=True)
torch.cuda.synchronize()
print("synced", out.status.cpu().numpy(), out.iterations.cpu().numpy(), flush=True)
