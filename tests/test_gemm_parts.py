"""Host-side check of the balanced (stream-K) GEMM partition rule the C-ABI
documents (include/ppd_b200.h ppd_gemm_parts): brute-force the ranges each
slot owns and compare the per-tile valid-slice count and each range's slice
index with the closed form the device consumers use."""
import random

import paper_2603_13358_b200 as ppd


def brute(tiles, kbt, slots):
    total = tiles * kbt
    touching = [[] for _ in range(tiles)]
    for c in range(slots):
        b0, b1 = c * total // slots, (c + 1) * total // slots
        for t in {x // kbt for x in range(b0, b1)}:
            touching[t].append(c)
    return touching


def test_partition_rule_matches_bruteforce():
    rng = random.Random(0)
    for _ in range(300):
        tiles = rng.randint(1, 60)
        kbt = rng.randint(1, 70)
        slots = rng.randint(1, min(160, tiles * kbt))
        g = ppd.GemmParts(n=0, kbt=kbt, slots=slots, rows=128, bn=256, n_tiles_t=1, total=tiles * kbt, stride=0)
        touching = brute(tiles, kbt, slots)
        for t in range(tiles):
            first = g.owner(t * kbt)
            assert touching[t] == list(range(first, first + len(touching[t])))  # slice j = c - first
            assert g.valid(t * 128, 0) == len(touching[t])


def test_uniform_parts_all_valid():
    g = ppd.GemmParts(n=3, kbt=0, slots=148, rows=128, bn=256, n_tiles_t=1, total=1, stride=0)
    assert g.valid(5000, 17) == 3


def test_hybrid_partition_whole_waves_then_stream_k():
    """dp leading tiles are whole-K units (one slice); the tail follows the
    stream-K rule over tail_slots ranges (gemm_tc.cu Sched)."""
    rng = random.Random(1)
    for _ in range(200):
        slots = rng.randint(1, 80)
        tiles = rng.randint(1, 300)
        kbt = rng.randint(4, 70)
        dp = (tiles // slots) * slots
        if dp == tiles:
            continue
        tslots = rng.randint(1, min(slots, (tiles - dp) * kbt))
        g = ppd.GemmParts(n=0, kbt=kbt, slots=tslots, rows=128, bn=256, n_tiles_t=1,
                          total=(tiles - dp) * kbt, stride=0, dp=dp)
        touching = brute(tiles - dp, kbt, tslots)
        for t in range(tiles):
            want = 1 if t < dp else len(touching[t - dp])
            assert g.valid(t * 128, 0) == want
