"""NEXT-3 timing: GPU LSH matching of one cfg3 batch's history tokens (32 x 640) against the 10^5
prototype library (product API only). python profiles/semlib_timing.py -> one JSON line."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import rcgen  # noqa: E402
from paper_2605_07443_b200.build import build  # noqa: E402
from paper_2605_07443_b200.api import RcContext  # noqa: E402

build()
wl = rcgen.CFG3
tiny = rcgen.CFG1.shape
W = rcgen.gen_weights(tiny, device=torch.device("cuda", 0))
ctx = RcContext(tiny, W, item_rows=64, hist_rows=1, prefix_rows=8, arena_rows=256, max_seq_len=256, max_batch_tokens=256)
protos = rcgen.gen_protos(wl)
cat = rcgen.gen_catalog(wl)
reqs = rcgen.gen_requests(wl, cat, protos, 32)
H = np.random.default_rng(5).standard_normal((128, 64)).astype(np.float32)
ctx.semlib_build(protos.token, protos.canon_pos - wl.prefix_len, protos.n_buckets, H, seed=11)
tok = torch.from_numpy(np.concatenate([r.hist_tokens for r in reqs]).astype(np.int32)).cuda()
off = torch.from_numpy(np.concatenate([np.arange(len(r.hist_tokens)) for r in reqs]).astype(np.int32)).cuda()
for _ in range(3):
    ctx.semlib_match(tok, off)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
reps = 20
for _ in range(reps):
    pid, cos = ctx.semlib_match(tok, off)
b.record()
torch.cuda.synchronize()
ms = a.elapsed_time(b) / reps
print(json.dumps({"what": "rc_semlib_match, cfg3 batch-32 history tokens vs 1e5 prototypes", "queries": tok.numel(),
                  "prototypes": int(protos.n), "ms": ms, "queries_per_s": tok.numel() / ms * 1e3,
                  "exact_match_frac": float((cos - 1.0).abs().lt(1e-6).float().mean())}))
ctx.close()
