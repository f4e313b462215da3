"""K8 decode layer kernel at small shapes (tiny config, a Qwen-style shape
with QKV bias and GQA group 5) against the CPU oracle, and its exclusivity
rule: a second device handle on the same GPU switches steps back to the
per-op kernels (K8's grid barrier needs every SM). Kept apart from
test_gpu_layer_kernel.py, whose module-scoped Llama-shape device would
otherwise still be open on the GPU."""
import numpy as np
import pytest

import paper_2603_13358_b200 as ppd
from oracle import oracle as O
from test_gpu_layer_kernel import check_vs_oracle, knob, launches

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def restore():
    knob(1)  # K8 is an option (default off): these tests exercise it
    yield
    knob(0)


def test_tiny_and_qwen_bias_shapes(gpu):
    for cfg, seed in ((ppd.tiny_cfg(), 5), (ppd.ModelCfg(3, 640, 5, 1, 128, 1280, 2048, 1e-6, 1e6, 1), 6)):
        dev = ppd.Device(0, cfg, max_step_tokens=4096, max_step_seqs=64)
        dev.load_random_weights(seed)
        dev.kv_pool_init(64 * 8)
        model = O.Model(O.cfg_from(cfg), seed)
        pool = O.KvPool(O.cfg_from(cfg), 64 * 8)
        rng = np.random.default_rng(seed)
        B = 40
        bts = np.arange(B * 8, dtype=np.int32).reshape(B, 8)
        q = rng.integers(20, 60, B).astype(np.int32)
        toks = rng.integers(0, cfg.vocab, int(q.sum())).astype(np.int32)
        # a prefill step (> 256 rows: per-op path) fills the caches, then decode steps take K8
        r, _ = check_vs_oracle(dev, model, pool, q, np.zeros(B, np.int32), toks, bts, 2e-2)
        ctx, tok = q.copy(), r.tokens
        for k in range(3):
            rr, n = launches(dev, [1] * B, ctx, tok, bts)
            assert n == 2 * cfg.n_layers + 7
            # replay the same step through the checker
            r2, _ = check_vs_oracle(dev, model, pool, [1] * B, ctx, tok, bts, 2e-2)
            assert (r2.tokens == rr.tokens).all()
            tok, ctx = r2.tokens, ctx + 1
        dev.close()


def test_second_device_on_the_gpu_disables_layer_kernel(gpu):
    """Two nodes on one GPU: K8's grid barrier needs all SMs, so steps fall
    back to the per-op kernels while both are open."""
    cfg = ppd.tiny_cfg()
    a = ppd.Device(0, cfg, max_step_tokens=64, max_step_seqs=8)
    a.load_random_weights(1)
    a.kv_pool_init(16)
    bts = np.arange(16, dtype=np.int32).reshape(2, 8)
    toks = np.array([5, 6], np.int32)
    _, n = launches(a, [1, 1], [3, 4], toks, bts)
    assert n == 2 * cfg.n_layers + 7
    b = ppd.Device(0, cfg, max_step_tokens=64, max_step_seqs=8)
    _, n = launches(a, [1, 1], [3, 4], toks, bts)
    assert n == 9 * cfg.n_layers + 4
    b.close()
    _, n = launches(a, [1, 1], [3, 4], toks, bts)
    assert n == 2 * cfg.n_layers + 7
    a.close()
