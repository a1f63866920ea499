import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np, torch
from paper_2512_23049_b200 import _native as nat
from paper_2512_23049_b200.config import ModelConfig
import test_gpu_kernels as T
hd, H, Hk = 128, 32, 8
rng = np.random.default_rng(11)
cfg = ModelConfig(n_layers=2, n_heads=H, n_kv_heads=Hk, head_dim=hd)
cache, lens = T._random_cache(cfg, rng, 8, dtype=torch.bfloat16)
calls = []
for a in range(6):
    own = 8 + a; n = int(rng.integers(1, 150))
    cache.register_message(own, "decoded", 0); cache.reserve_slots(own, [1] * n); cache.log_append(own, 0, n)
    parents = [int(p) for p in rng.permutation(8)[:int(rng.integers(0, 7))]]
    calls.append((own, parents, [n - 1]))
print("calls", calls)
out, (rt_d, vis, blk, items, rpo, rp, counts) = T._assemble(cache, calls, 16, 2, 0)
R = len(out["row_t"]); pl_ = out["plan"]; n_items = pl_.n_items
tab, par, off = [], [], 0
for own, parents, ts in calls:
    tab += [own, len(par), len(parents), off, len(ts)]; par += parents; off += len(ts)
dev = lambda a: torch.tensor(a, dtype=torch.int32, device="cuda")
fat = torch.full((n_items, 64), -9, dtype=torch.int32, device="cuda")
s = torch.cuda.current_stream().cuda_stream
nat.assemble(cache.msg_len.dev.data_ptr(), cache.msg_pt.dev.data_ptr(), cache.page_table.dev.data_ptr(),
             dev(tab).data_ptr(), dev(par + [0]).data_ptr(), len(calls), rt_d.data_ptr(), R, None, 0, 64, 16, 2,
             vis[0].data_ptr(), vis[1].data_ptr(), vis[2].data_ptr(), blk.data_ptr(), items.data_ptr(),
             rpo.data_ptr(), rp.data_ptr(), counts.data_ptr(), pl_.n_vis, pl_.n_blk_rows, n_items, pl_.n_parts, 0,
             fat.data_ptr(), s)
torch.cuda.synchronize()
print("counts", counts.tolist(), "n_items", n_items)
print("items", items.cpu().tolist())
print("fat[:3]", fat[:3].cpu().tolist())
print("rpo", rpo.tolist(), "rp", rp.tolist())
q = torch.randn(R, H, hd, device="cuda")
po = torch.zeros(pl_.n_parts, H, hd, device="cuda"); pl = torch.full((pl_.n_parts, H), 7.0, device="cuda")
cnt = torch.zeros(R * Hk, dtype=torch.int32, device="cuda")
o2 = torch.zeros(2 * R, H * hd, dtype=torch.bfloat16, device="cuda")
nat.decode_attn(q.data_ptr(), cache.k_pool.data_ptr(), cache.v_pool.data_ptr(), 1, Hk, cache.n_pages, 64, H, hd,
                fat.data_ptr(), counts.data_ptr(), n_items, rpo.data_ptr(), rp.data_ptr(), po.data_ptr(), pl.data_ptr(),
                cnt.data_ptr(), o2.data_ptr(), 1, R, 3, 0, s)
torch.cuda.synchronize()
print("lse", pl[:, ::8].tolist())
oc = torch.zeros(2 * R, H * hd, dtype=torch.bfloat16, device="cuda")
nat.attn_combine(po.data_ptr(), pl.data_ptr(), rpo.data_ptr(), rp.data_ptr(), R, H, hd, oc.data_ptr(), nat.BF16, 1, s)
torch.cuda.synchronize()
print("fused rows abs", (o2[:R].float().abs().sum(1)).tolist())
print("combine rows abs", (oc[:R].float().abs().sum(1)).tolist())
for trial in range(4):
    fatp = fat.data_ptr() if trial % 2 else None
    tab_d, par_d = dev(tab), dev(par + [0])
    nat.assemble(cache.msg_len.dev.data_ptr(), cache.msg_pt.dev.data_ptr(), cache.page_table.dev.data_ptr(),
                 tab_d.data_ptr(), par_d.data_ptr(), len(calls), rt_d.data_ptr(), R, None, 0, 64, 16, 2,
                 vis[0].data_ptr(), vis[1].data_ptr(), vis[2].data_ptr(), blk.data_ptr(), items.data_ptr(),
                 rpo.data_ptr(), rp.data_ptr(), counts.data_ptr(), 1000, 1000, 1000, 1000, 0, fatp, s)
    torch.cuda.synchronize()
    print("trial", trial, "counts", counts.tolist(), "plan", (pl_.n_vis, pl_.n_items, pl_.n_parts))
print("msg_len dev", cache.msg_len.dev[:16].tolist(), "host", cache.msg_len.host[:16].tolist())
