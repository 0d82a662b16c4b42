"""Host-link probe: H2D / D2H bandwidth of pinned buffers at the bench's output size (734 MB), one copy vs
split across streams, so that bench.py's e2e number can be read against the link it runs on."""
import time

import torch


def bw(nbytes, fn, reps=5):
    fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return nbytes * reps / (time.perf_counter() - t) / 1e9


def main():
    n = 16384 * 11200
    d = torch.empty(n, device="cuda")
    h = torch.empty(n).pin_memory()
    print(f"D2H 1 copy : {bw(4 * n, lambda: h.copy_(d, non_blocking=True)):.1f} GB/s")
    print(f"H2D 1 copy : {bw(4 * n, lambda: d.copy_(h, non_blocking=True)):.1f} GB/s")
    for k in (2, 4):
        ss = [torch.cuda.Stream() for _ in range(k)]
        ch = n // k

        def split():
            for i, s in enumerate(ss):
                with torch.cuda.stream(s):
                    h[i * ch:(i + 1) * ch].copy_(d[i * ch:(i + 1) * ch], non_blocking=True)
        print(f"D2H {k} streams: {bw(4 * n, split):.1f} GB/s")

    def both():
        s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
        with torch.cuda.stream(s1):
            h.copy_(d, non_blocking=True)
        with torch.cuda.stream(s2):
            d.copy_(h, non_blocking=True)
    print(f"D2H+H2D concurrent (per direction): {bw(4 * n, both):.1f} GB/s")
    import subprocess
    print(subprocess.run(["nvidia-smi", "--query-gpu=pcie.link.gen.current,pcie.link.width.current,pcie.link.gen.max",
                          "--format=csv"], capture_output=True, text=True).stdout)


if __name__ == "__main__":
    main()
