#!/usr/bin/env python
"""e2e tuning: raw pinned H2D/D2H copy bandwidth vs the host-resident push pipeline
at several chunk sizes (BORIS_HOST_CHUNK is read when the pipeline is created)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import torch  # noqa: E402


def copy_bw(nbytes, direction):
    h = torch.empty(nbytes // 4, dtype=torch.float32, pin_memory=True)
    d = torch.empty(nbytes // 4, dtype=torch.float32, device="cuda")
    for _ in range(2):
        (d.copy_(h, non_blocking=True) if direction == "h2d" else h.copy_(d, non_blocking=True))
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(5):
        (d.copy_(h, non_blocking=True) if direction == "h2d" else h.copy_(d, non_blocking=True))
    b.record()
    torch.cuda.synchronize()
    return 5 * nbytes / (a.elapsed_time(b) * 1e-3) / 1e9


def main():
    for mb in (16, 256, 1024):
        print(json.dumps({"exp": "pinned_copy", "mbytes": mb,
                          "h2d_gbs": copy_bw(mb << 20, "h2d"), "d2h_gbs": copy_bw(mb << 20, "d2h")}),
              flush=True)
    for chunk in (1 << 20, 4 << 20, 16 << 20):
        env = dict(os.environ, BORIS_HOST_CHUNK=str(chunk))
        out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--particles",
                              "100000000", "--steps", "5", "--warmup", "3", "--e2e-steps", "4",
                              "--no-cpu-baseline"], capture_output=True, text=True, env=env).stdout
        line = json.loads(out.strip().splitlines()[-1])
        e2e = line["e2e"]
        print(json.dumps({"exp": "e2e_chunk", "chunk": chunk, "e2e_updates_per_s": e2e["value"],
                          "ms_per_step": e2e["ms_per_step"],
                          "h2d_gbs_effective": e2e["h2d_bytes_per_step"] / e2e["ms_per_step"] / 1e6}),
              flush=True)


if __name__ == "__main__":
    main()
