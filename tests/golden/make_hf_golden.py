"""Pin the transformer oracle to an independent implementation:
transformers.LlamaForCausalLM (5.5, fp32, eager attention) loaded with the
same seeded bf16 weights the GPU and oracle/llama_ref.c generate.

Run in the build container (transformers + torch CPU are installed there):
    python tests/golden/make_hf_golden.py
Writes tests/golden/hf_<config>.npz with, for the seeded prompt:
    tokens      int32 [T]
    logits      fp32 [vocab]   next-token logits at position T-1
    k, v        fp32 [L, n_kv, P, hd]  K (after RoPE) and V at sample positions P
    pos         int64 [P]
tests/test_oracle_pinned.py checks both CPU oracles against these files.

TEST INFRASTRUCTURE ONLY (the product never imports transformers).
"""
from __future__ import annotations

import os
import sys

import numpy as np
import torch

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

import llama_np  # noqa: E402

CONFIGS = {
    # name: (dims, T) — dims = (L, H, n_heads, n_kv_heads, head_dim, ffn, vocab)
    "tiny": ((2, 256, 4, 4, 64, 1024, 32000), 2048),
    "gqa8_hd128": ((2, 1024, 16, 2, 128, 2048, 32768), 1024),
}
WEIGHT_SEED, PROMPT_SEED = 1234, 42


def hf_model(dims):
    from transformers import LlamaConfig, LlamaForCausalLM

    L, H, nh, nkv, hd, F, V = dims
    cfg = LlamaConfig(vocab_size=V, hidden_size=H, intermediate_size=F, num_hidden_layers=L,
                      num_attention_heads=nh, num_key_value_heads=nkv, head_dim=hd, rms_norm_eps=1e-5,
                      rope_theta=500000.0, max_position_embeddings=8192, tie_word_embeddings=False,
                      attention_bias=False, mlp_bias=False, attn_implementation="eager")
    m = LlamaForCausalLM(cfg).float().eval()
    ref = llama_np.LlamaNp(dims, 1, seed=WEIGHT_SEED)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a))  # noqa: E731
    with torch.no_grad():
        m.model.embed_tokens.weight.copy_(t(llama_np.weight(WEIGHT_SEED, llama_np.TID_EMBED, V, H, 1.0)))
        m.lm_head.weight.copy_(t(llama_np.weight(WEIGHT_SEED, llama_np.TID_LMHEAD, V, H, ref.s_h)))
        m.model.norm.weight.fill_(1.0)
        for l, layer in enumerate(m.model.layers):
            w = ref.layer(l)
            layer.self_attn.q_proj.weight.copy_(t(w["q"]))
            layer.self_attn.k_proj.weight.copy_(t(w["k"]))
            layer.self_attn.v_proj.weight.copy_(t(w["v"]))
            layer.self_attn.o_proj.weight.copy_(t(w["o"]))
            layer.mlp.gate_proj.weight.copy_(t(w["g"]))
            layer.mlp.up_proj.weight.copy_(t(w["u"]))
            layer.mlp.down_proj.weight.copy_(t(w["d"]))
            layer.input_layernorm.weight.fill_(1.0)
            layer.post_attention_layernorm.weight.fill_(1.0)
    return m


def main():
    from paper_2410_03065_b200.cake import Cake

    for name, (dims, T) in CONFIGS.items():
        toks = Cake().token_stream(PROMPT_SEED, T).astype(np.int32)
        m = hf_model(dims)
        with torch.no_grad():
            out = m(torch.from_numpy(toks.astype(np.int64))[None], use_cache=True)
        logits = out.logits[0, -1].numpy().astype(np.float32)
        pos = np.array(sorted({0, 1, 63, T // 2, T - 2, T - 1}), dtype=np.int64)
        cache = out.past_key_values
        ks, vs = [], []
        for l in range(dims[0]):
            lay = cache.layers[l]
            ks.append(lay.keys[0][:, pos].numpy())    # [n_kv, P, hd]
            vs.append(lay.values[0][:, pos].numpy())
        path = os.path.join(HERE, f"hf_{name}.npz")
        np.savez_compressed(path, tokens=toks, logits=logits, k=np.stack(ks).astype(np.float32),
                            v=np.stack(vs).astype(np.float32), pos=pos, dims=np.array(dims), T=T,
                            weight_seed=WEIGHT_SEED, prompt_seed=PROMPT_SEED)
        print(name, path, "top1", int(logits.argmax()), os.path.getsize(path), "bytes")


if __name__ == "__main__":
    main()
