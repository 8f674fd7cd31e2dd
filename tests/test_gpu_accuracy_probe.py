"""bf16 error budget at full depth (diagnostic, opt-in: RC_ACCURACY_PROBE=1).

Llama-3-8B shape, all 32 layers, one 1024-token prompt prefilled in full (every position FORCED,
no prefix) through librc, and through a plain torch bf16 model (cuBLAS GEMMs + SDPA; once with a
bf16 residual stream as in stock bf16 inference, once with an fp32 residual stream as librc keeps
it), each against the fp64 oracle O-FULL. Prints rel-L2 of K per layer (error growth with depth),
of the final hidden states and of the last-token logits. It tells whether the selective path's
~0.9% at cfg3 is the bf16 floor of this random-init model or an excess of the kernels.
"""
import json
import os

import numpy as np
import pytest
import torch

import rcgen
from oracle.model import OracleModel, full_prefill
from oracle.numerics import bf16_to_f32
from tests.helpers import rel_l2

pytestmark = [pytest.mark.gpu, pytest.mark.slow,
              pytest.mark.skipif(os.environ.get("RC_ACCURACY_PROBE") != "1", reason="opt-in diagnostic")]

N_TOK = 1024


def _torch_bf16(W, shape, tokens, fp32_residual):
    import torch.nn.functional as F
    dev = W["embed"].device
    n = tokens.shape[0]
    H, Hk, dh = shape.n_heads, shape.n_kv_heads, shape.head_dim
    inv = 1.0 / (shape.rope_theta ** (torch.arange(0, dh, 2, device=dev, dtype=torch.float64) / dh))
    ang = torch.arange(n, device=dev, dtype=torch.float64)[:, None] * inv[None]
    cos, sin = ang.cos().float(), ang.sin().float()

    def rope(x):  # [h, n, dh] fp32
        x0, x1 = x[..., :dh // 2], x[..., dh // 2:]
        return torch.cat([x0 * cos - x1 * sin, x1 * cos + x0 * sin], -1)

    def rms(x, g):
        xf = x.float()
        return (xf * torch.rsqrt(xf.pow(2).mean(-1, keepdim=True) + shape.rms_eps) * g.float()).to(torch.bfloat16)

    Ks = []
    with torch.no_grad():
        x = W["embed"][tokens].float() if fp32_residual else W["embed"][tokens]
        for lw in W["layers"]:
            a = rms(x, lw["ln1"])
            q = rope((a @ lw["wq"].T).float().view(n, H, dh).transpose(0, 1)).to(torch.bfloat16)
            k = rope((a @ lw["wk"].T).float().view(n, Hk, dh).transpose(0, 1)).to(torch.bfloat16)
            v = (a @ lw["wv"].T).view(n, Hk, dh).transpose(0, 1)
            Ks.append(k.transpose(0, 1).float().cpu().numpy())
            o = F.scaled_dot_product_attention(q[None], k[None], v[None], is_causal=True, enable_gqa=True)[0]
            o = o.transpose(0, 1).reshape(n, H * dh)
            x = x + (o @ lw["wo"].T).to(x.dtype)
            m = rms(x, lw["ln2"])
            h = (F.silu((m @ lw["wg"].T).float()) * (m @ lw["wu"].T).float()).to(torch.bfloat16)
            x = x + (h @ lw["wd"].T).to(x.dtype)
        logits = rms(x[-1:], W["norm"]).float() @ W["lm_head"].float().T
    return x.float().cpu().numpy(), logits[0].cpu().numpy(), Ks


def test_bf16_error_budget_full_depth():
    from paper_2605_07443_b200.build import build
    from tests import gpu_helpers as G
    from tests.helpers import make_case, oracle_pools
    build()
    wl = rcgen.CFG2
    shape = wl.shape
    dev = torch.device("cuda", 0)
    W = rcgen.gen_weights(shape, seed=0, device=dev)
    Wh = {"embed": W["embed"].cpu(), "norm": W["norm"].cpu(), "lm_head": W["lm_head"].cpu(),
          "layers": [{k: v.cpu() for k, v in lw.items()} for lw in W["layers"]]}
    case = make_case(wl, weights=Wh)
    pools = oracle_pools(case)
    ctx, _ = G.make_ctx(case, pools, N_TOK, Wd=W)
    lay = G.gpu_layouts(ctx, case)[0]
    lay = dict(lay, tokens=lay["tokens"][:N_TOK].copy(), cls=np.full(N_TOK, 1, np.uint8),
               src_id=lay["src_id"][:N_TOK].copy(), src_off=lay["src_off"][:N_TOK].copy())
    seqs = ctx.assemble([lay], prefix_id=G.PREFIX_ID, gather_from=1)
    out = ctx.selective_prefill(seqs, 10000, 10000, check_layer=1, hidden=True, n_cand=len(lay["cand_idtok"]))
    torch.cuda.synchronize()
    ours_x = out["hidden"].cpu().numpy()
    ours_logits = out["logits"][0].cpu().numpy()
    ours_K = [bf16_to_f32(ctx.read_kv(seqs[0], l, N_TOK)[0].cpu().numpy().view(np.uint16))
              for l in range(shape.n_layers)]
    ctx.release(seqs)
    ctx.close()
    tok = torch.tensor(lay["tokens"].astype(np.int64), device=dev)
    tb = _torch_bf16(W, shape, tok, fp32_residual=False)
    tf = _torch_bf16(W, shape, tok, fp32_residual=True)
    ref = full_prefill(OracleModel(shape, Wh), lay["tokens"].tolist())
    rep = {}
    for name, (x, lg, Ks) in {"librc": (ours_x, ours_logits, ours_K), "torch_bf16_residual": tb,
                              "torch_fp32_residual": tf}.items():
        rep[name] = {"hidden": rel_l2(x, ref["x"]), "logits": rel_l2(lg, ref["logits_last"]),
                     "K_by_layer": [round(rel_l2(Ks[l], ref["K"][l]), 5) for l in range(shape.n_layers)]}
    print("accuracy probe", json.dumps(rep))
    os.makedirs("gpurun_out", exist_ok=True)
    with open(os.path.join("gpurun_out", "accuracy_probe.json"), "w") as f:
        json.dump(rep, f, indent=1)
    assert rep["librc"]["logits"] <= 1.5 * rep["torch_fp32_residual"]["logits"] + 1e-3
