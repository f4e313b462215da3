"""Pins the numerics oracle (oracle/model_oracle.c) to a PUBLISHED decoder
implementation: HF transformers 5.5.0 `LlamaForCausalLM` / `Qwen2ForCausalLM`
(eager attention, fp32 on CPU) loaded with the same counter-hash random
weights the device fill kernels and the oracle generate (mo_weight_bf16).

For each case it runs a two-turn conversation through the HF model — turn 1
(full prefill), turn 2 (new tokens appended), then greedy decode steps fed
with HF's own argmax — and stores, per step the oracle will replay, the fp32
logits of the step's last position (full vocabulary rows, float16 for the
large-vocabulary case to keep the fixture small), HF's greedy id and its
top-1/top-2 margin. tests/test_oracle.py replays the same token stream
through the oracle (prefill, append over the paged cache, decode) and
compares.

The reference (/root/reference) has no model; this is the
published implementation the "Llama-3-8B-shape" / "Qwen2.5-32B-shape" of
BASELINE.json refers to. Conventions mapped onto HF:
  q/k/v/o, gate/up/down, embed, lm_head = hash tensors 1..8 (logical [out][in]
  = nn.Linear.weight); Qwen q/k/v biases = hash tensors 9..11; all RMSNorm
  weights 1; untied lm_head; rotate-half RoPE (HF's default rope_type).

Run (CPU, ~1 min, ~12 GB RAM):  python tests/golden/make_hf_fixtures.py
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np
import torch

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
from oracle import oracle as O  # noqa: E402

# tensor ids of model_oracle.h
T_EMBED, T_WQ, T_WK, T_WV, T_WO, T_WGATE, T_WUP, T_WDOWN, T_LMHEAD, T_BQ, T_BK, T_BV = range(12)

CASES = {
    # name: (cfg tuple = n_layers, d_model, Hq, Hkv, head_dim, d_ff, vocab, eps, theta, qkv_bias), seed,
    #       turn-1 tokens, turn-2 tokens, decode steps, logits dtype
    "tiny_llama": ((2, 512, 4, 1, 128, 1024, 2048, 1e-5, 5e5, 0), 20260313, 64, 32, 6, "float32"),
    "tiny_qwen": ((2, 640, 5, 1, 128, 1280, 2048, 1e-6, 1e6, 1), 77, 45, 30, 4, "float32"),
    "llama8b_2layer": ((2, 4096, 32, 8, 128, 14336, 128256, 1e-5, 5e5, 0), 20260313, 48, 16, 3, "float16"),
}


def bf16_tensor(seed, tensor, layer, shape):
    n = int(np.prod(shape))
    return torch.from_numpy(O.bf16_to_f32(O.tensor_bf16(seed, tensor, layer, n)).reshape(shape).copy())


def hf_model(cfg, seed):
    L, d, Hq, Hkv, Dh, F, V, eps, theta, bias = cfg
    kw = dict(vocab_size=V, hidden_size=d, intermediate_size=F, num_hidden_layers=L, num_attention_heads=Hq,
              num_key_value_heads=Hkv, head_dim=Dh, rms_norm_eps=eps, rope_theta=theta,
              max_position_embeddings=8192, tie_word_embeddings=False, attn_implementation="eager")
    if bias:
        from transformers import Qwen2Config, Qwen2ForCausalLM
        conf = Qwen2Config(**kw)
        model = Qwen2ForCausalLM(conf)
    else:
        from transformers import LlamaConfig, LlamaForCausalLM
        conf = LlamaConfig(**kw)
        model = LlamaForCausalLM(conf)
    qd, kd = Hq * Dh, Hkv * Dh
    sd = {"model.embed_tokens.weight": bf16_tensor(seed, T_EMBED, 0, (V, d)),
          "lm_head.weight": bf16_tensor(seed, T_LMHEAD, 0, (V, d)),
          "model.norm.weight": torch.ones(d)}
    for l in range(L):
        p = f"model.layers.{l}."
        sd[p + "self_attn.q_proj.weight"] = bf16_tensor(seed, T_WQ, l, (qd, d))
        sd[p + "self_attn.k_proj.weight"] = bf16_tensor(seed, T_WK, l, (kd, d))
        sd[p + "self_attn.v_proj.weight"] = bf16_tensor(seed, T_WV, l, (kd, d))
        sd[p + "self_attn.o_proj.weight"] = bf16_tensor(seed, T_WO, l, (d, qd))
        sd[p + "mlp.gate_proj.weight"] = bf16_tensor(seed, T_WGATE, l, (F, d))
        sd[p + "mlp.up_proj.weight"] = bf16_tensor(seed, T_WUP, l, (F, d))
        sd[p + "mlp.down_proj.weight"] = bf16_tensor(seed, T_WDOWN, l, (d, F))
        sd[p + "input_layernorm.weight"] = torch.ones(d)
        sd[p + "post_attention_layernorm.weight"] = torch.ones(d)
        if bias:
            sd[p + "self_attn.q_proj.bias"] = bf16_tensor(seed, T_BQ, l, (qd,))
            sd[p + "self_attn.k_proj.bias"] = bf16_tensor(seed, T_BK, l, (kd,))
            sd[p + "self_attn.v_proj.bias"] = bf16_tensor(seed, T_BV, l, (kd,))
    missing, unexpected = model.load_state_dict(sd, strict=False)
    missing = [k for k in missing if "rotary" not in k]
    assert not missing and not unexpected, (missing, unexpected)
    return model.eval()


def make_case(name, cfg, seed, n1, n2, n_dec, ldtype):
    torch.manual_seed(0)
    model = hf_model(cfg, seed)
    V = cfg[6]
    rng = np.random.default_rng(list(CASES).index(name) + 1)
    turn1 = rng.integers(0, V, n1).tolist()
    turn2 = rng.integers(0, V, n2).tolist()
    # steps replayed by the oracle: (q_len, ctx, tokens) -> logits of the last position
    steps = [(n1, 0, turn1)]
    ids = turn1 + turn2
    steps.append((n2, n1, turn2))
    logits, greedy, margin = [], [], []
    with torch.no_grad():
        out = model(torch.tensor([ids]), use_cache=True)
        past = out.past_key_values
        full = out.logits[0].float()
        for row in (n1 - 1, n1 + n2 - 1):
            logits.append(full[row].numpy())
        nxt = int(torch.argmax(full[-1]))
        for _ in range(n_dec):
            steps.append((1, len(ids), [nxt]))
            ids.append(nxt)
            out = model(torch.tensor([[nxt]]), past_key_values=past, use_cache=True)
            past = out.past_key_values
            lg = out.logits[0, -1].float()
            logits.append(lg.numpy())
            nxt = int(torch.argmax(lg))
    for lg in logits:
        top2 = np.sort(lg)[-2:]
        greedy.append(int(np.argmax(lg)))
        margin.append(float(top2[1] - top2[0]))
    arr = np.stack(logits).astype(ldtype)
    path = os.path.join(HERE, f"hf_{name}.npz")
    np.savez_compressed(path, logits=arr, greedy=np.array(greedy, dtype=np.int32),
                        margin=np.array(margin, dtype=np.float32),
                        q_len=np.array([s[0] for s in steps], dtype=np.int32),
                        ctx=np.array([s[1] for s in steps], dtype=np.int32),
                        tokens=np.array([t for s in steps for t in s[2]], dtype=np.int32),
                        cfg=np.array(cfg[:7], dtype=np.int64), eps_theta=np.array(cfg[7:9], dtype=np.float64),
                        qkv_bias=np.array(cfg[9]), seed=np.array(seed, dtype=np.uint64))
    return {"case": name, "steps": len(steps), "file": os.path.basename(path),
            "bytes": os.path.getsize(path), "greedy": greedy}


def main():
    import transformers
    torch.set_num_threads(os.cpu_count() or 1)
    meta = {"generator": "tests/golden/make_hf_fixtures.py", "transformers": transformers.__version__,
            "torch": torch.__version__, "dtype": "float32 (eager attention)", "cases": []}
    for name, spec in CASES.items():
        if len(sys.argv) > 1 and name not in sys.argv[1:]:
            continue
        info = make_case(name, *spec)
        print(json.dumps(info))
        meta["cases"].append(info)
    with open(os.path.join(HERE, "hf_fixtures.json"), "w") as f:
        json.dump(meta, f, indent=1)


if __name__ == "__main__":
    main()
