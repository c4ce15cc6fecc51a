"""One Morton pack and unpack at 256^3 (for ncu)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_1511_06029_b200 as q  # noqa: E402

g = torch.randn(1 << 24, dtype=torch.float64, device="cuda")
x = q.morton_pack(g, 3, 8)
back = q.morton_unpack(x, 3, 8)
torch.cuda.synchronize()
assert torch.equal(back.view(-1), g)
print("ok")
