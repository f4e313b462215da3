"""§8f-3: the routing gateway fronting GPU workers that EXECUTE the routed
turns. The gateway (engine/gateway.cpp, the reference's wire protocol and
routing, reference gateway.cpp:94-255) decides each turn; the workers are
device handles with their own paged KV pools on the GPU:

* route "P_path": the prefill worker recomputes the whole history into a
  temporary block table (ppd_step), then the missing tokens are copied to the
  pinned decode worker's pool (ppd_kv_copy, reference simulator.cpp:349-353);
* route "D_local": the decode worker appends the new tokens over its cache
  (ppd_step with ctx = cached tokens);
* either way the decode worker samples the turn's output tokens.

Checked: both routes occur; each conversation stays on the decode backend the
gateway pinned; the decode worker's cached-context report drives the next
route request; every generated token equals the CPU oracle's greedy token
wherever the oracle's top-1/top-2 margin is clear (routing moves work between
GPUs/pools, never the tokens)."""
import json

import numpy as np
import pytest

import paper_2603_13358_b200 as ppd
from oracle import oracle as O
from paper_2603_13358_b200 import engine as E

pytestmark = pytest.mark.gpu

MARGIN = 0.05
SEED = 99
BT = 16


class Worker:
    """A GPU worker: one device handle (one node), its KV pool, a block allocator."""

    def __init__(self, role, cfg, gpu=0, blocks=256):
        self.role = role
        self.dev = ppd.Device(gpu, cfg, max_step_tokens=1024, max_step_seqs=16)
        self.dev.load_random_weights(SEED)
        self.dev.kv_pool_init(blocks)
        self.free = list(range(blocks))
        self.tables = {}  # key -> block list
        self.tokens = {}  # key -> cached tokens

    def ensure(self, key, n_tokens):
        t = self.tables.setdefault(key, [])
        while len(t) * BT < n_tokens:
            t.append(self.free.pop(0))
        return t

    def release(self, key):
        self.free.extend(self.tables.pop(key, []))
        self.tokens.pop(key, None)

    def run(self, key, q, ctx, toks):
        t = self.ensure(key, ctx + len(toks))
        r = self.dev.step([len(toks)], [ctx], np.asarray(toks, np.int32), np.asarray([t], np.int32))
        self.tokens[key] = ctx + len(toks)
        return int(r.tokens[0])

    def close(self):
        self.dev.close()


def route(gw, conv, turn, n_in, n_ctx, n_out, now):
    msg = {"kind": "route", "conv_first_message": conv, "turn_index": turn, "new_input_tokens": n_in,
           "cached_context_tokens": n_ctx, "target_output_tokens": n_out}
    return json.loads(gw.handle(json.dumps(msg), now))


def test_gateway_routes_turns_executed_on_gpu_workers(gpu):
    cfg = ppd.tiny_cfg()
    gw = E.Gateway({"x": 0.5})
    workers = {}
    now = 0.0
    for role, addr in (("P", "gpu0/p"), ("D", "gpu0/d0"), ("D", "gpu0/d1")):
        rep = json.loads(gw.handle(json.dumps({"kind": "register", "role": role, "address": addr, "gpu": 0}), now))
        workers[rep["id"]] = Worker(role, cfg)
    model = O.Model(O.cfg_from(cfg), SEED)
    rng = np.random.default_rng(4)
    hist = {}      # conv -> full token history (inputs + outputs)
    pinned = {}    # conv -> decode backend id
    routes = []
    checked = 0
    try:
        for turn in (1, 2, 3):
            for c in range(4):
                conv = f"conversation-{c}"
                now += 0.01
                for b in workers:
                    gw.handle(json.dumps({"kind": "heartbeat", "id": b}), now)
                new = rng.integers(0, cfg.vocab, int(rng.integers(20, 41))).tolist()
                n_out = 6
                h = hist.setdefault(conv, [])
                d_id = pinned.get(conv)
                cached = workers[d_id].tokens.get(conv, 0) if d_id is not None else 0
                rep = route(gw, conv, turn, len(new), cached, n_out, now)
                assert rep["ok"], rep
                d_id = rep["decode_backend"]
                if conv in pinned:
                    assert d_id == pinned[conv]  # session affinity
                pinned[conv] = d_id
                D = workers[d_id]
                assert D.role == "D" and rep["decode_gpu"] == 0
                routes.append(rep["target"])
                h.extend(new)
                if rep["target"] == "P_path":
                    P = workers[rep["prefill_backend"]]
                    assert P.role == "P" and rep["prefill_gpu"] == 0
                    key = f"tmp-{conv}-{turn}"
                    first = P.run(key, len(h), 0, h)                     # full recompute on P
                    have = D.tokens.get(conv, 0)
                    D.ensure(conv, len(h))
                    ppd.kv_copy(P.dev, D.dev, np.asarray(P.tables[key], np.int32),
                                np.asarray(D.tables[conv], np.int32), have, len(h) - have)
                    D.tokens[conv] = len(h)
                    P.release(key)
                else:  # append over D's cache: the previous turn's last output token + the new input
                    c0 = D.tokens[conv]
                    first = D.run(conv, len(h) - c0, c0, h[c0:])
                out = [first]
                for _ in range(n_out - 1):
                    out.append(D.run(conv, 1, len(h) + len(out) - 1, [out[-1]]))
                # the oracle replays the conversation's full history (prefill) and the decode steps
                pool = O.KvPool(O.cfg_from(cfg), 64)
                bt = np.arange(64, dtype=np.int32)[None]
                t_o, _, m = model.step(pool, [len(h)], [0], np.asarray(h, np.int32), bt)
                ref, margins = [int(t_o[0])], [float(m[0])]
                for k in range(n_out - 1):
                    t_o, _, m = model.step(pool, [1], [len(h) + k], np.asarray([out[k]], np.int32), bt)
                    ref.append(int(t_o[0]))
                    margins.append(float(m[0]))
                for g, r_, mg in zip(out, ref, margins):
                    if mg > MARGIN:
                        assert g == r_, (conv, turn, out, ref, margins)
                        checked += 1
                # the output tokens join the history; the last one's KV is written by the next step
                h.extend(out)
                D.tokens[conv] = len(h) - 1
        st = json.loads(gw.handle('{"kind":"stats"}', now))
        assert "P_path" in routes and "D_local" in routes
        assert st["queries"] == 12 and st["p_path"] == routes.count("P_path")
        assert len(set(pinned.values())) == 2  # round robin over the two decode workers
        assert checked >= 24
    finally:
        for w in workers.values():
            w.close()
        gw.close()
