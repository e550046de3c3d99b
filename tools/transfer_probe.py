"""Host link / NVLink copy rates on the GPU box (CUDA-event timed), the
denominators of bench.py's step_roofline (PCIE_H2D_GBS / PCIE_D2H_GBS):

  python tools/transfer_probe.py > profiles/r02_transfer_probe.json

pinned H2D, D2H, both directions at once (two streams), and peer-to-peer
device copies over NVLink when more than one device is visible."""
import json

import torch


def timed(fn, reps=5):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn()
    torch.cuda.synchronize()
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps * 1e-3


def main():
    out = {"device": torch.cuda.get_device_name(0), "devices": torch.cuda.device_count()}
    for gib in (1, 4):
        n = gib << 30
        h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
        h2 = torch.empty(n, dtype=torch.uint8, pin_memory=True)
        d = torch.empty(n, dtype=torch.uint8, device="cuda")
        d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
        t_h2d = timed(lambda: d.copy_(h, non_blocking=True))
        t_d2h = timed(lambda: h.copy_(d, non_blocking=True))
        s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

        def both():
            with torch.cuda.stream(s1):
                d.copy_(h, non_blocking=True)
            with torch.cuda.stream(s2):
                h2.copy_(d2, non_blocking=True)
            torch.cuda.current_stream().wait_stream(s1)
            torch.cuda.current_stream().wait_stream(s2)
        t_bi = timed(both)
        out[f"{gib}GiB"] = {"h2d_gbs": round(n / t_h2d / 1e9, 2), "d2h_gbs": round(n / t_d2h / 1e9, 2),
                            "bidir_total_gbs": round(2 * n / t_bi / 1e9, 2)}
        del h, h2, d, d2
    if torch.cuda.device_count() > 1:
        n = 1 << 30
        a = torch.empty(n, dtype=torch.uint8, device="cuda:0")
        b = torch.empty(n, dtype=torch.uint8, device="cuda:1")
        t = timed(lambda: b.copy_(a, non_blocking=True))
        out["p2p_0_to_1_gbs"] = round(n / t / 1e9, 2)
    else:
        out["p2p"] = "one device visible (gpurun leases 1 GPU): NVLink not measurable here"
    print(json.dumps(out))


if __name__ == "__main__":
    main()
