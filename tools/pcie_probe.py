"""Pinned host <-> device copy rates on this box (the bound of the e2e numbers):
H2D alone, D2H alone, both at once (separate streams)."""
import time

import torch


def rate(fn, nbytes, reps=3):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        t = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t)
    return round(nbytes / best / 1e9, 1)


def main():
    n = 4 << 30
    h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    h2 = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(n, dtype=torch.uint8, device="cuda")
    d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    print("H2D GB/s", rate(lambda: d.copy_(h, non_blocking=True), n))
    print("D2H GB/s", rate(lambda: h2.copy_(d2, non_blocking=True), n))

    def both():
        with torch.cuda.stream(s1):
            d.copy_(h, non_blocking=True)
        with torch.cuda.stream(s2):
            h2.copy_(d2, non_blocking=True)
    print("H2D+D2H concurrent, GB/s each way", rate(both, n))


if __name__ == "__main__":
    main()
