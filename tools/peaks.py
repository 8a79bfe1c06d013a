"""Host-link and cuBLAS DGEMM peaks on the B200 box (companion to fp64_peak.cu).

Prints one JSON line per measurement.  Run under gpurun; nothing here is on the
product path.
"""
import json

import torch


def time_ms(fn, reps=5):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(reps):
        s.record()
        fn()
        e.record()
        e.synchronize()
        best = min(best, s.elapsed_time(e))
    return best


def main():
    dev = torch.device("cuda:0")
    for n in (4096, 8192):
        a = torch.randn(n, n, dtype=torch.float64, device=dev)
        b = torch.randn(n, n, dtype=torch.float64, device=dev)
        ms = time_ms(lambda: torch.matmul(a, b))
        print(json.dumps({"what": "cublas_dgemm", "n": n, "ms": ms, "tflops": 2 * n**3 / ms / 1e9}))
    # rotation-shaped DGEMM: Z^T (1000x1000) x X (1000 x 100000)
    z = torch.randn(1000, 1000, dtype=torch.float64, device=dev)
    x = torch.randn(100000, 1000, dtype=torch.float64, device=dev)
    ms = time_ms(lambda: torch.matmul(x, z))
    print(json.dumps({"what": "cublas_dgemm_rotation", "shape": [1000, 1000, 100000], "ms": ms,
                      "tflops": 2 * 1000 * 1000 * 100000 / ms / 1e9}))
    del x
    nbytes = 1 << 30
    h = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    d = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    ms = time_ms(lambda: d.copy_(h, non_blocking=True))
    print(json.dumps({"what": "h2d_pinned", "bytes": nbytes, "gbs": nbytes / ms / 1e6}))
    ms = time_ms(lambda: h.copy_(d, non_blocking=True))
    print(json.dumps({"what": "d2h_pinned", "bytes": nbytes, "gbs": nbytes / ms / 1e6}))
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    h2 = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    d2 = torch.empty(nbytes, dtype=torch.uint8, device=dev)

    def both():
        with torch.cuda.stream(s1):
            d.copy_(h, non_blocking=True)
        with torch.cuda.stream(s2):
            h2.copy_(d2, non_blocking=True)
        torch.cuda.current_stream().wait_stream(s1)
        torch.cuda.current_stream().wait_stream(s2)

    ms = time_ms(both)
    print(json.dumps({"what": "h2d+d2h_concurrent", "bytes_each": nbytes, "gbs_each": nbytes / ms / 1e6}))


if __name__ == "__main__":
    main()
