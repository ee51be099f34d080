"""Where the e2e step goes: pinned H2D of theta/phi alone, D2H of z alone,
the device iteration alone, and H2D concurrent with the iteration (the
configs[3] bench workload at N = 1)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1505_03851_b200 as wd  # noqa: E402
from paper_1505_03851_b200.device_lda import DeviceLDA  # noqa: E402


def ev():
    return torch.cuda.Event(enable_timing=True)


def main():
    args = bench.parse()
    dev = torch.device("cuda", 0)
    off, words, base = bench.make_shard(torch, 0, 1, args, dev)
    dc = wd.DeviceCorpus.from_csr(off, words, doc_base=base, vocab_size=args.vocab)
    lda = DeviceLDA(dc, args.topics, args.vocab, seed=args.seed)
    lda.init_uniform()
    for t in range(3):
        lda.iterate(t)
    th_h = lda.theta.cpu().pin_memory()
    ph_h = lda.phi.cpu().pin_memory()
    z_h = torch.empty(lda.z.numel(), dtype=torch.int16).pin_memory()
    th_d = torch.empty_like(lda.theta)
    up = torch.cuda.Stream()
    down = torch.cuda.Stream()
    st = torch.cuda.current_stream()
    out = {}
    torch.cuda.synchronize()
    a, b = ev(), ev()
    a.record(up)
    with torch.cuda.stream(up):
        th_d.copy_(th_h, non_blocking=True)
    b.record(up)
    torch.cuda.synchronize()
    out["h2d_theta_alone_ms"] = a.elapsed_time(b)
    a, b = ev(), ev()
    a.record(st)
    lda.iterate(10)
    b.record(st)
    torch.cuda.synchronize()
    out["iteration_alone_ms"] = a.elapsed_time(b)
    z16 = lda.z.to(torch.int16)
    a, b = ev(), ev()
    a.record(down)
    with torch.cuda.stream(down):
        z_h.copy_(z16, non_blocking=True)
    b.record(down)
    torch.cuda.synchronize()
    out["d2h_z16_alone_ms"] = a.elapsed_time(b)
    # H2D concurrent with an iteration
    up.wait_stream(st)
    a, b, c, d = ev(), ev(), ev(), ev()
    a.record(up)
    with torch.cuda.stream(up):
        th_d.copy_(th_h, non_blocking=True)
    b.record(up)
    c.record(st)
    lda.iterate(11)
    d.record(st)
    torch.cuda.synchronize()
    out["h2d_theta_during_iteration_ms"] = a.elapsed_time(b)
    out["iteration_during_h2d_ms"] = c.elapsed_time(d)
    # H2D concurrent with D2H
    a, b, c, d = ev(), ev(), ev(), ev()
    a.record(up)
    with torch.cuda.stream(up):
        th_d.copy_(th_h, non_blocking=True)
    b.record(up)
    c.record(down)
    with torch.cuda.stream(down):
        z_h.copy_(z16, non_blocking=True)
    d.record(down)
    torch.cuda.synchronize()
    out["h2d_theta_with_d2h_ms"] = a.elapsed_time(b)
    out["d2h_with_h2d_ms"] = c.elapsed_time(d)
    out["theta_bytes"] = th_h.numel() * 4
    print(json.dumps(out))


if __name__ == "__main__":
    main()
