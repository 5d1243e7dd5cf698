"""syn256 SCORE determinism probe: the same device-generated link walks scored
on the device twice and through the host entry (chunked), compared bit for
bit; mismatching rows re-scored alone.  python tools/syn256_determinism.py [B]"""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2406_01566_b200 as h  # noqa: E402
from paper_2406_01566_b200 import clusters  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 2_000_000
d = clusters.CONFIGS["syn256-120l"]("float")
c = h.Cluster.from_json(json.dumps(d))
e = h.Engine(c)
e.mode = "score"
N = e.num_nodes
dev = torch.device("cuda:0")
sp = torch.cuda.current_stream().cuda_stream
pl = torch.empty((B, N, 2), dtype=torch.int16, device=dev)
e.generate_walk_device(20240611, 0, B, pl.data_ptr(), sp)
torch.cuda.synchronize()


def dev_score():
    v = torch.empty(B, dtype=torch.float64, device=dev)
    st = torch.empty(B, dtype=torch.int32, device=dev)
    e.score_device(pl.data_ptr(), B, v.data_ptr(), st.data_ptr(), True, sp)
    torch.cuda.synchronize()
    return v.cpu().numpy(), st.cpu().numpy()


v1, s1 = dev_score()
v2, s2 = dev_score()
host = torch.empty((B, N, 2), dtype=torch.int16, pin_memory=True)
host.copy_(pl)
hv = torch.empty(B, dtype=torch.float64, pin_memory=True)
hs = torch.empty(B, dtype=torch.int32, pin_memory=True)
e.score_best_host_ptr(host.data_ptr(), B, hv.data_ptr(), hs.data_ptr(), True)
v3 = hv.numpy()
b1, b2, b3 = (x.view(np.int64) for x in (v1, v2, v3))
d12 = np.nonzero(b1 != b2)[0]
d13 = np.nonzero(b1 != b3)[0]
print("device vs device mismatches", len(d12), d12[:10])
print("device vs host mismatches", len(d13), d13[:10])
for i in list(d12[:5]) + list(d13[:5]):
    rv = [e.score(host.numpy()[i:i + 1])[0][0] for _ in range(3)]
    print(i, v1[i], v2[i], v3[i], "alone:", rv, "status", s1[i], s2[i])
