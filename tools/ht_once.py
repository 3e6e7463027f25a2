"""One config-4 batched hSVD truncation (batch 64), device-resident, for ncu."""
import sys
import torch
sys.path.insert(0, ".")
from paper_1803_10270_b200 import _lib, workloads  # noqa: E402

w = workloads.cfg4(0, batch=64)
d, Q, k, nb = w["d"], w["Q"], w["k"], w["frames"].shape[0]
dev = torch.device("cuda")
F = torch.as_tensor(w["frames"]).to(dev)
B = torch.as_tensor(w["transfers"]).to(dev)
ro = 16
OF = torch.zeros((nb, d, Q, ro), dtype=torch.float64, device=dev)
OB = torch.zeros((nb, d - 1, ro, ro, ro), dtype=torch.float64, device=dev)
ranks = torch.zeros((nb, 2 * d - 1), dtype=torch.int32, device=dev)
est = torch.zeros(nb, dtype=torch.float64, device=dev)
norms = torch.zeros(nb, dtype=torch.float64, device=dev)
L = _lib.lib()
nbytes = L.tp_ht_truncate_ws_bytes(d, Q, k, nb)
ws = torch.empty(nbytes, dtype=torch.uint8, device=dev)
st = torch.cuda.current_stream().cuda_stream
s = L.tp_ht_truncate_f64(d, Q, k, nb, F.data_ptr(), B.data_ptr(), ro, 0.0, OF.data_ptr(), OB.data_ptr(),
                         ranks.data_ptr(), est.data_ptr(), norms.data_ptr(), ws.data_ptr(), ws.numel(), st)
torch.cuda.synchronize()
print("status", s)
