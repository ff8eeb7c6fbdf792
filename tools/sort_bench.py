"""Device time of the hand-written radix sort (radix.cu) on the step's two
sort shapes -- 26M (tile, slot) pairs with 15-bit keys (30 % equal "culled"
keys) and 4M depth keys (isg_sort_depth) -- against torch.sort (CUB) on the
same data, CUDA events, best of 5.

    python tools/sort_bench.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def timeit(fn, reps=5):
    import torch
    best = 1e30
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b))
    return best


def main():
    import torch
    from paper_2509_05216_b200 import _lib as L
    g = torch.Generator(device="cuda").manual_seed(0)
    n = 26_000_000
    tk = torch.randint(0, 16384, (n,), generator=g, device="cuda", dtype=torch.int32)
    tk[torch.rand(n, generator=g, device="cuda") < 0.3] = 16384
    tk = tk.to(torch.int16)
    tv = torch.arange(n, dtype=torch.int32, device="cuda")
    ws = L.Workspace()
    ko, vo = torch.empty_like(tk), torch.empty_like(tv)
    ours = timeit(lambda: L.sort_pairs(tk, tv, (0, 15), ws, ko, vo))
    ref = timeit(lambda: torch.sort(tk.to(torch.int32), stable=True))
    print(f"tiles 26M u16/15 bits: ours {ours:.3f} ms, torch.sort(int32) {ref:.3f} ms")
    m = 4_000_000
    depth = 100.0 + 400.0 * torch.rand(m, generator=g, device="cuda", dtype=torch.float64)
    dk = depth.view(torch.int64).clone()
    dk[:20000] = -1
    dv = torch.arange(m, dtype=torch.int32, device="cuda")
    ws2 = L.Workspace()
    k2, v2 = torch.empty_like(dk), torch.empty_like(dv)
    ours = timeit(lambda: L.sort_depth(dk, dv, ws2, k2, v2))
    ref = timeit(lambda: torch.sort(dk, stable=True))
    print(f"depth 4M u64: ours {ours:.3f} ms, torch.sort(int64) {ref:.3f} ms")


if __name__ == "__main__":
    main()
