"""Host-link micro-benchmark of the runtime's copy tiers: demand batches of
n Mixtral-8x7B experts through the native runtime, raw tier vs XC tier
(staging ring + decode stream), no compute.  Prints per-batch device time,
wire GB/s, the decode kernel's time alone and its per-segment time inside
the runtime (under the next segment's H2D copy)."""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

from paper_2510_10302_b200 import codec as X
from paper_2510_10302_b200.cache import ExpertId, NativeExpertCache
from paper_2510_10302_b200.model import fill_expert_blob, get_arch


def main(n_rows=12, batch=6, reps=4):
    a = get_arch("mixtral_8x7b")
    dev = torch.device("cuda", 0)
    stage = torch.empty((a.expert_elems,), dtype=torch.bfloat16, device=dev)
    enc = X.XcEncoder(X.expert_segments(a.ffn, a.hidden), dev)
    blobs, raws = [], []
    for r in range(n_rows):
        fill_expert_blob(stage, a, 1234, r)
        hdr = enc.plan(stage)
        blobs.append(enc.encode(stage, hdr).cpu())
        raws.append(stage.cpu())
    stride = (max(b.numel() for b in blobs) + 4095) // 4096 * 4096
    host_xc = torch.zeros((n_rows, stride), dtype=torch.uint8).pin_memory()
    for i, b in enumerate(blobs):
        host_xc[i, : b.numel()] = b
    host_raw = torch.stack(raws).pin_memory()
    E = n_rows  # one layer per "row": ids (l, 0..n_rows-1) over layers
    res = {}
    for tier in ("raw", "xc"):
        cap = batch * 2
        pool = torch.empty((cap, a.expert_elems), dtype=torch.bfloat16, device=dev)
        copy, dec = torch.cuda.Stream(), torch.cuda.Stream()
        host = host_raw if tier == "raw" else host_xc
        L = 64
        c = NativeExpertCache(cap, L, E, dev_pool_ptr=pool.data_ptr(), host_pool_ptr=host.data_ptr(),
                              host_index=[i % n_rows for i in range(L * E)], slot_bytes=a.expert_bytes,
                              copy_stream_ptr=copy.cuda_stream)
        staging = None
        if tier == "xc":
            staging = torch.empty((3 * stride,), dtype=torch.uint8, device=dev)
            c.set_codec(stride, staging.data_ptr(), stride, 3, dec.cuda_stream)
            c.decode_timing(True)
        cur = torch.cuda.current_stream()
        times = []
        for rep in range(reps + 1):
            ids = [ExpertId(rep % L, (rep * batch + j) % E) for j in range(batch)]
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record(cur)
            cur.wait_stream(copy)  # start together
            slots = c.demand_load(ids)
            for s in slots:
                c.wait_slot(s, cur.cuda_stream)
            e1.record(cur)
            for s in slots:
                c.mark_read(s, cur.cuda_stream)
            torch.cuda.synchronize()
            if rep:
                times.append(e0.elapsed_time(e1))
        if tier == "xc":
            st = c.decode_stats()  # segment decodes inside the runtime, each under the next segment's H2D
            res["decode_in_runtime_us_per_segment"] = st["ms"] * 1e3 / max(1, st["launches"])
            res["decode_in_runtime_gbs"] = st["gbs"]
        wire = c.wire_bytes()["demand"]
        log = c.transfer_log()
        ms = float(np.median(times))
        per_batch_wire = wire / (reps + 1)
        res[tier] = {"ms_per_batch": ms, "wire_gbs": per_batch_wire / (ms / 1e3) / 1e9,
                     "expert_gbs": batch * a.expert_bytes / (ms / 1e3) / 1e9,
                     "log_ms": [round(r["end_ms"] - r["start_ms"], 3) for r in log]}
        c.close()
        del pool, staging
    # decode alone
    hdr = X.header_at(host_xc[0].data_ptr())
    blob = host_xc[0, : int(hdr.blob_bytes)].to(dev)
    out = torch.empty((a.expert_elems,), dtype=torch.bfloat16, device=dev)
    X.decode(blob, hdr, out)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        X.decode(blob, hdr, out)
    e1.record()
    torch.cuda.synchronize()
    res["decode_ms"] = e0.elapsed_time(e1) / 10
    res["wire_ratio"] = float(np.mean([b.numel() for b in blobs])) / a.expert_bytes
    # plain H2D of one blob vs one raw expert
    for name, src in (("h2d_blob", host_xc[0, : int(hdr.blob_bytes)]), ("h2d_raw", host_raw[0])):
        d = torch.empty(src.shape, dtype=src.dtype, device=dev)
        e0.record()
        for _ in range(5):
            d.copy_(src, non_blocking=True)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 5
        res[name] = {"ms": ms, "gbs": src.numel() * src.element_size() / (ms / 1e3) / 1e9}
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
