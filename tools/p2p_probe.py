"""NVLink peer-copy probe (copy engines, one process driving every GPU):
unidirectional 0->1, bidirectional 0<->1, and the all-to-all pattern of the
co-located configs (every GPU sends to every other at once).  Reports GB/s
per GPU per direction: the reference for what the SM-driven pushes reach."""
import sys
import time

import torch


def run(pairs, nbytes, reps=5):
    n = torch.cuda.device_count()
    bufs = {}
    streams = {}
    for (a, b) in pairs:
        bufs[(a, b)] = (torch.empty(nbytes, dtype=torch.uint8, device=f"cuda:{a}"),
                        torch.empty(nbytes, dtype=torch.uint8, device=f"cuda:{b}"))
        streams[(a, b)] = torch.cuda.Stream(device=f"cuda:{a}")
    for d in range(n):
        torch.cuda.synchronize(d)
    best = 1e9
    for _ in range(reps):
        t0 = time.perf_counter()
        for k, (src, dst) in bufs.items():
            with torch.cuda.stream(streams[k]):
                dst.copy_(src, non_blocking=True)
        for d in range(n):
            torch.cuda.synchronize(d)
        best = min(best, time.perf_counter() - t0)
    tx = {}
    for (a, b) in pairs:
        tx[a] = tx.get(a, 0) + nbytes
    return {a: round(v / best / 1e9, 1) for a, v in tx.items()}, round(best * 1e3, 2)


def main():
    n = torch.cuda.device_count()
    nb = int(float(sys.argv[1]) * 2**30) if len(sys.argv) > 1 else 2**31
    print("uni 0->1", run([(0, 1)], nb))
    print("bidi 0<->1", run([(0, 1), (1, 0)], nb))
    if n >= 4:
        allp = [(a, b) for a in range(n) for b in range(n) if a != b]
        print(f"all-to-all {n}", run(allp, nb // (n - 1)))
        print("fan-out 0->1,2,3", run([(0, 1), (0, 2), (0, 3)], nb // 3))


if __name__ == "__main__":
    main()
