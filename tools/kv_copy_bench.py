"""K7 KV-transfer throughput on one GPU (P and D pools on the same device, so
HBM -> HBM: every byte is read once and written once): ppd_kv_copy of `need`
tokens (Llama-3-8B shape, 131,072 B/token) at block-aligned and unaligned
starts. Reports GB/s of transferred KV (the metric) and the HBM traffic rate
(2x). PPD_LIB=<path> A/Bs another build."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_13358_b200 as ppd  # noqa: E402


def main():
    if os.environ.get("PPD_LIB"):
        ppd._lib = ppd.load_lib(os.environ["PPD_LIB"], strict=False)
    cfg = ppd.llama8b_cfg()
    kvb = ppd.kv_block_bytes(cfg) // 16
    nblk = 1200
    devs = []
    for _ in range(2):
        d = ppd.Device(0, cfg, max_step_tokens=64, max_step_seqs=8)
        d.kv_pool_init(nblk)
        devs.append(d)
    src, dst = devs
    rng = np.random.default_rng(0)
    for start, need in ((0, 1536), (2053, 1536), (0, 8192), (4101, 8192)):
        nb = (start + need + 15) // 16
        bs = rng.permutation(nblk)[:nb].astype(np.int32)
        bd = rng.permutation(nblk)[:nb].astype(np.int32)
        ppd.kv_copy(src, dst, bs, bd, start, need)
        ms = [ppd.kv_copy(src, dst, bs, bd, start, need) for _ in range(20)]
        t = float(np.median(ms))
        gbs = need * kvb / (t * 1e-3) / 1e9
        print(json.dumps({"start": start, "need": need, "ms": t, "kv_gbs": gbs, "hbm_traffic_gbs": 2 * gbs}), flush=True)
    for d in devs:
        d.close()


if __name__ == "__main__":
    main()
