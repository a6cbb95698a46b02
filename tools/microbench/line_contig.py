# A/B: the line kernel on contiguous lines (1D plan, non-tiled path) vs the 2D passes
import torch, paper_1802_10291_b200 as mci
def t(fn, n=20):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    a.record()
    for _ in range(n): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / n
bank = [("identity",), ("derivative", 1)]
p = mci.Plan(2, 512, 2048, bank)
for rows in (32768, 65536):
    g = torch.randn(rows, 2, 512, device="cuda")
    f = torch.empty(rows, 2048, device="cuda")
    print("1D contiguous rows", rows, "ms", round(t(lambda: p.execute(g, f)), 4), "launches", p.launches(rows))
p2 = mci.Plan2D(2, 512, bank, 2, 512, bank, 4)
g2 = torch.randn(64, 2, 2, 512, 512, device="cuda")
o2 = torch.empty(64, 2048, 2048, device="cuda")
print("2D 64 images ms", round(t(lambda: p2.execute(g2, o2)), 4))
