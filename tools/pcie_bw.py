"""Raw pinned host<->device copy bandwidth on this box (the e2e path's bound).

python tools/pcie_bw.py   -> H2D, D2H and both directions at once, GB/s
"""
import torch


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps / 1000.0


def main():
    n = 717 << 20  # the bench scene's bytes per step
    h = torch.empty(n, dtype=torch.uint8).pin_memory()
    h2 = torch.empty(n, dtype=torch.uint8).pin_memory()
    d = torch.empty(n, dtype=torch.uint8, device="cuda")
    d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    t_h2d = timed(lambda: d.copy_(h, non_blocking=True))
    t_d2h = timed(lambda: h2.copy_(d2, non_blocking=True))

    def both():
        with torch.cuda.stream(s1):
            d.copy_(h, non_blocking=True)
        with torch.cuda.stream(s2):
            h2.copy_(d2, non_blocking=True)
        torch.cuda.current_stream().wait_stream(s1)
        torch.cuda.current_stream().wait_stream(s2)
    t_both = timed(both)
    print(f"H2D {n / t_h2d / 1e9:.1f} GB/s  D2H {n / t_d2h / 1e9:.1f} GB/s  "
          f"concurrent {2 * n / t_both / 1e9:.1f} GB/s total ({t_both * 1e3:.2f} ms for {n >> 20} MiB each way)")


if __name__ == "__main__":
    main()
