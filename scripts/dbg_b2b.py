"""Debug: which outputs differ between serialised and back-to-back fused decodes."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
sys.path.insert(0, "tests")
sys.path.insert(0, "oracle")
import test_gpu_decode as T

shapes = [(4, 8, 32), (3, 4, 4)]
ctxs = [[40, 300, 17], [64, 1]]
split = int(sys.argv[1]) if len(sys.argv) > 1 else 0


def run(mode):
    cache, groups = T.build_pool(shapes, ctxs, seed=5, phys_layers=1)
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    torch.cuda.set_stream(s)
    cache.set_stream(s)
    b = cache.batch(groups)
    gen = torch.Generator(device="cuda").manual_seed(11)
    res = []
    for step in range(2):
        b.grow(1)
        cache.flush()
        ks = [[(torch.rand((len(ids), 1, H, 128), generator=gen, device="cuda") - 0.5).half() for (mi, ids), (L, H, Hq) in zip(groups, shapes)] for _ in range(4)]
        vs = [[(torch.rand((len(ids), 1, H, 128), generator=gen, device="cuda") - 0.5).half() for (mi, ids), (L, H, Hq) in zip(groups, shapes)] for _ in range(4)]
        qs = [[torch.randn((len(ids), Hq, 128), generator=gen, device="cuda").half() for (mi, ids), (L, H, Hq) in zip(groups, shapes)] for _ in range(4)]
        outs = [[torch.full_like(q, float("nan")) for q in ql] for ql in qs]
        for layer in range(4):
            b.decode(qs[layer], outs[layer], layer, split_tokens=split, k=ks[layer], v=vs[layer])
            if mode == "sync":
                torch.cuda.synchronize()
        torch.cuda.synchronize()
        res.append([[o.clone() for o in ol] for ol in outs])
    torch.cuda.synchronize()
    torch.cuda.set_stream(torch.cuda.default_stream())
    return T.host_image(cache), res


a_img, a = run("sync")
b_img, b = run("eager")
print("pool equal", np.array_equal(a_img, b_img))
for st in range(2):
    for layer in range(4):
        for g in range(2):
            x, y = a[st][layer][g], b[st][layer][g]
            if not torch.equal(x, y):
                d = (x.float() - y.float()).abs()
                bad = torch.nonzero(torch.isnan(d) | (d > 0))
                reqs = sorted(set(bad[:, 0].tolist()))
                heads = sorted(set(bad[:, 1].tolist()))
                print(f"step {st} layer {layer} group {g}: diff reqs {reqs} heads {heads[:12]}.. max {torch.nan_to_num(d, nan=99).max().item()} nan_sync {torch.isnan(x).any().item()} nan_eager {torch.isnan(y).any().item()}")
