"""NVLink evidence for the slab-transpose / record-exchange push (k_push,
wsb_push_blocks) in ONE process (so ncu can profile it): every GPU pushes
a block into every other GPU's memory over NVLink (peer access), as the
multi-GPU driver's symmetric-memory pushes do. Prints one JSON line:
per-GPU push bandwidth (CUDA events on the pushing stream) for one peer and
for all peers at once.

    python tools/nvlink_push_probe.py [--mib 256]"""
import argparse
import ctypes as C
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402
from cuda.bindings import runtime as cudart  # noqa: E402

from paper_2504_00959_b200 import _lib as L  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mib", type=int, default=256)
    ap.add_argument("--reps", type=int, default=10)
    a = ap.parse_args()
    n = torch.cuda.device_count()
    assert n >= 2, "needs >= 2 GPUs"
    for i in range(n):
        cudart.cudaSetDevice(i)
        for j in range(n):
            if i != j:
                cudart.cudaDeviceEnablePeerAccess(j, 0)
    nbytes = a.mib << 20
    src = [torch.empty(nbytes, dtype=torch.uint8, device=f"cuda:{i}").fill_(i + 1) for i in range(n)]
    # dst[j][i]: GPU j's receive block from GPU i
    dst = [[torch.empty(nbytes, dtype=torch.uint8, device=f"cuda:{j}") for _ in range(n)] for j in range(n)]
    ctx, streams = [], []
    for i in range(n):
        with torch.cuda.device(i):
            s = torch.cuda.Stream(i)
            c = L.Context(i)
            c.bind_stream(s.cuda_stream)
            ctx.append(c)
            streams.append(s)
    lib = L.lib()

    def push(i, peers):
        srcs = (C.c_void_p * len(peers))(*[src[i].data_ptr()] * len(peers))
        dsts = (C.c_void_p * len(peers))(*[dst[j][i].data_ptr() for j in peers])
        sizes = (C.c_int64 * len(peers))(*[nbytes] * len(peers))
        L.check(lib.wsb_push_blocks(ctx[i].handle, len(peers), srcs, dsts, sizes))

    out = {"gpus": n, "block_mib": a.mib}
    # one peer: GPU 0 -> GPU 1
    with torch.cuda.device(0):
        for _ in range(2):
            push(0, [1])
        torch.cuda.synchronize(0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(streams[0])
        for _ in range(a.reps):
            push(0, [1])
        e1.record(streams[0])
        torch.cuda.synchronize(0)
        ms = e0.elapsed_time(e1) / a.reps
    out["one_peer_GBps"] = round(nbytes / (ms / 1e3) / 1e9, 1)
    # all-to-all: every GPU pushes to all peers at once
    for i in range(n):
        push(i, [j for j in range(n) if j != i])
    for i in range(n):
        torch.cuda.synchronize(i)
    evs = []
    for i in range(n):
        with torch.cuda.device(i):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(streams[i])
            evs.append((e0, e1))
    for _ in range(a.reps):
        for i in range(n):
            with torch.cuda.device(i):
                push(i, [j for j in range(n) if j != i])
    for i in range(n):
        with torch.cuda.device(i):
            evs[i][1].record(streams[i])
    for i in range(n):
        torch.cuda.synchronize(i)
    ms = max(e0.elapsed_time(e1) for e0, e1 in evs) / a.reps
    out["all_to_all_per_gpu_out_GBps"] = round((n - 1) * nbytes / (ms / 1e3) / 1e9, 1)
    out["all_to_all_aggregate_GBps"] = round(n * (n - 1) * nbytes / (ms / 1e3) / 1e9, 1)
    # correctness: every received block holds its sender's bytes
    ok = all(int(dst[j][i][:16].float().mean().item()) == i + 1 for j in range(n) for i in range(n) if i != j)
    out["blocks_correct"] = ok
    out["note"] = ("k_push: 16-byte stores into peer memory (NVLink), CUDA events on each pushing "
                   "GPU's stream; NVLink 5 is 900 GB/s per direction per GPU")
    print(json.dumps(out))


if __name__ == "__main__":
    main()
