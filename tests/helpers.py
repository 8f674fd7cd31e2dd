"""Test-side helpers: build oracle inputs from the seeded generators, HF reference models."""
import numpy as np
import torch

import rcgen
from oracle.layout import layout_from_request, classify_tokens


def make_case(wl, n_req=1, start=0, device="cpu", weights=None):
    """Generator outputs for `n_req` requests of workload `wl` (CPU tensors)."""
    shape = wl.shape
    cat = rcgen.gen_catalog(wl)
    protos = rcgen.gen_protos(wl)
    sys_tok = rcgen.gen_system_prompt(wl)
    reqs = rcgen.gen_requests(wl, cat, protos, n_req, start)
    W = weights if weights is not None else rcgen.gen_weights(shape)
    return dict(wl=wl, shape=shape, cat=cat, protos=protos, sys=sys_tok, reqs=reqs, W=W)


def oracle_pools(case, reqs=None, prefix_kv=None):
    """Pool dicts for oracle.assemble holding exactly the blocks the requests touch."""
    wl, shape = case["wl"], case["shape"]
    reqs = reqs if reqs is not None else case["reqs"]
    items = sorted({int(i) for r in reqs for i in r.cand_items})
    protos = sorted({int(p) for r in reqs for p in r.hist_protos})
    ikv = rcgen.pools.item_kv(shape, wl.item_len, items)
    hq, hs = rcgen.pools.hist_kv(shape, protos)
    pkv = prefix_kv if prefix_kv is not None else rcgen.pools.prefix_kv(shape, wl.prefix_len)
    item_d = {it: (ikv[j], wl.prefix_len) for j, it in enumerate(items)}
    hist_d = {pi: (hq[j].numpy(), hs[j].numpy(), int(case["protos"].canon_pos[pi]))
              for j, pi in enumerate(protos)}
    return dict(items=item_d, hist=hist_d, prefix=pkv, item_ids=items, proto_ids=protos,
                item_kv=ikv, hist_q=hq, hist_s=hs)


def layouts(case, reqs=None):
    reqs = reqs if reqs is not None else case["reqs"]
    return [layout_from_request(r, case["cat"], case["sys"]) for r in reqs]


def hf_model(shape, W):
    """HF transformers LlamaForCausalLM / Qwen2ForCausalLM (fp32, CPU) with the same weights."""
    from transformers import LlamaConfig, LlamaForCausalLM, Qwen2Config, Qwen2ForCausalLM
    common = dict(vocab_size=shape.vocab, hidden_size=shape.d_model, intermediate_size=shape.d_ff,
                  num_hidden_layers=len(W["layers"]), num_attention_heads=shape.n_heads,
                  num_key_value_heads=shape.n_kv_heads, rms_norm_eps=shape.rms_eps,
                  rope_theta=shape.rope_theta, max_position_embeddings=16384,
                  tie_word_embeddings=False)
    if shape.qkv_bias:
        cfg = Qwen2Config(**common)
        cls = Qwen2ForCausalLM
    else:
        cfg = LlamaConfig(head_dim=shape.head_dim, attention_bias=False, mlp_bias=False, **common)
        cls = LlamaForCausalLM
    cfg._attn_implementation = "eager"
    model = cls(cfg).float().eval()
    sd = {"model.embed_tokens.weight": W["embed"], "model.norm.weight": W["norm"],
          "lm_head.weight": W["lm_head"]}
    for l, lw in enumerate(W["layers"]):
        p = f"model.layers.{l}."
        sd[p + "input_layernorm.weight"] = lw["ln1"]
        sd[p + "post_attention_layernorm.weight"] = lw["ln2"]
        for a, b in (("wq", "q_proj"), ("wk", "k_proj"), ("wv", "v_proj"), ("wo", "o_proj")):
            sd[p + f"self_attn.{b}.weight"] = lw[a]
        if shape.qkv_bias:
            for a, b in (("bq", "q_proj"), ("bk", "k_proj"), ("bv", "v_proj")):
                sd[p + f"self_attn.{b}.bias"] = lw[a]
        for a, b in (("wg", "gate_proj"), ("wu", "up_proj"), ("wd", "down_proj")):
            sd[p + f"mlp.{b}.weight"] = lw[a]
    sd = {k: v.float() for k, v in sd.items()}
    missing, unexpected = model.load_state_dict(sd, strict=False)
    assert not unexpected and all("rotary" in m for m in missing), (missing, unexpected)
    return model


def rel_l2(a, b):
    a = np.asarray(a, dtype=np.float64).ravel()
    b = np.asarray(b, dtype=np.float64).ravel()
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def assert_top10_ranking(gpu_scores, ref_scores, logit_err):
    """R19 / north star "identical top-10 candidate ranking": rank = score desc, ties -> lower slot.
    logit_err = the measured RMS error of the request's logits (GPU vs oracle). Wherever the
    oracle's gap between its i-th and (i+1)-th candidate exceeds 4 logit_err, the GPU's top-(i+1)
    set must equal the oracle's (near-ties may swap). Returns the number of positions checked."""
    g = np.asarray(gpu_scores, dtype=np.float64)
    r = np.asarray(ref_scores, dtype=np.float64)
    order_r = sorted(range(len(r)), key=lambda i: (-r[i], i))
    order_g = sorted(range(len(g)), key=lambda i: (-g[i], i))
    checked = 0
    for i in range(min(10, len(r) - 1)):
        if r[order_r[i]] - r[order_r[i + 1]] > 4 * logit_err:
            assert set(order_g[:i + 1]) == set(order_r[:i + 1]), (i, order_g[:11], order_r[:11], logit_err)
            checked += 1
    return checked


def rms_err(a, b):
    a = np.asarray(a, dtype=np.float64).ravel()
    b = np.asarray(b, dtype=np.float64).ravel()
    return float(np.sqrt(np.mean((a - b) ** 2)))
