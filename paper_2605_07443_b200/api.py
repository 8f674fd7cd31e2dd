"""Thin Python face of librc (same names as include/rc.h, argument marshalling only).

PyTorch provides device memory and streams; every computation of the hot path happens in
librc's sm_100a kernels. Nothing here imports oracle/.
"""
import ctypes as C

import numpy as np
import torch

from . import _lib as R
from ._lib import check, lib, np_ptr


def _stream(stream):
    if stream is None:
        stream = torch.cuda.current_stream()
    return C.c_void_p(stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream))


def _dptr(t):
    return C.c_void_p(t.data_ptr()) if t is not None else C.c_void_p(0)


def _ptr_array(tensors):
    arr = (C.c_void_p * len(tensors))(*[t.data_ptr() for t in tensors])
    return C.cast(arr, R.PP), arr


class RcContext:
    """rc_create/rc_destroy around one device. `weights`: rcgen naming, bf16 CUDA tensors."""

    def __init__(self, shape, weights, item_rows, hist_rows, prefix_rows, arena_rows, max_seq_len, max_batch_tokens,
                 remote_rows=0, device=0, host_item_rows=0):
        lib()
        self.shape = shape
        self.device = device
        self._keep = [weights]
        md = R.ModelDesc(shape.n_layers, shape.d_model, shape.n_heads, shape.n_kv_heads, shape.head_dim, shape.d_ff,
                         shape.vocab, float(shape.rope_theta), float(shape.rms_eps), int(shape.qkv_bias))
        w = R.Weights()
        w.embed, w.final_norm, w.lm_head = (weights[k].data_ptr() for k in ("embed", "norm", "lm_head"))
        for name in ("ln1", "wq", "wk", "wv", "wo", "ln2", "wg", "wu", "wd") + (("bq", "bk", "bv") if shape.qkv_bias else ()):
            p, arr = _ptr_array([lw[name] for lw in weights["layers"]])
            self._keep.append(arr)
            setattr(w, name, p)
        pd = R.PoolDesc(item_rows, remote_rows, hist_rows, prefix_rows, arena_rows, max_seq_len, max_batch_tokens,
                        host_item_rows)
        out = C.c_void_p()
        check(lib().rc_create(C.byref(md), C.byref(w), C.byref(pd), device, C.byref(out)))
        self.ctx = out
        self.max_batch_tokens = max_batch_tokens
        self.arena_rows = arena_rows

    def close(self):
        if getattr(self, "ctx", None):
            lib().rc_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # interpreter shutdown: module globals may already be gone
            pass

    # ------------------------------------------------------------------ pools
    def pool_register_blocks(self, kind, ids, n_tokens, canon_pos, kv, scales=None, stream=None):
        ids = np.ascontiguousarray(ids, dtype=np.uint64)
        nt = np.ascontiguousarray(n_tokens, dtype=np.int32)
        cp = np.ascontiguousarray(canon_pos, dtype=np.int32)
        assert kv.is_cuda and kv.is_contiguous()
        check(lib().rc_pool_register_blocks(self.ctx, kind, len(ids), np_ptr(ids, C.c_uint64), np_ptr(nt, C.c_int32),
                                            np_ptr(cp, C.c_int32), _dptr(kv), _dptr(scales), _stream(stream)))

    def pool_contains(self, kind, ids):
        ids = np.ascontiguousarray(ids, dtype=np.uint64)
        out = np.zeros(len(ids), np.uint8)
        check(lib().rc_pool_contains(self.ctx, kind, len(ids), np_ptr(ids, C.c_uint64), np_ptr(out, C.c_uint8)))
        return out.astype(bool)

    def pool_locate(self, ids):
        ids = np.ascontiguousarray(ids, dtype=np.uint64)
        out = np.zeros(len(ids), np.int64)
        check(lib().rc_pool_locate(self.ctx, len(ids), np_ptr(ids, C.c_uint64), np_ptr(out, C.c_int64)))
        return out

    # ------------------------------------------------------------------ requests
    @staticmethod
    def decompose_prompt(prefix_tokens, hist_proto, hist_tokens, cand_item, cand_tokens, tail_tokens):
        pt = np.ascontiguousarray(prefix_tokens, np.int32)
        hp = np.ascontiguousarray(hist_proto, np.int64)
        ht = np.ascontiguousarray(hist_tokens, np.int32)
        ci = np.ascontiguousarray(cand_item, np.int64)
        cl = np.ascontiguousarray([len(t) for t in cand_tokens], np.int32)
        ct = np.ascontiguousarray(np.concatenate([np.asarray(t, np.int32) for t in cand_tokens]) if len(cand_tokens)
                                  else np.zeros(0, np.int32))
        tt = np.ascontiguousarray(tail_tokens, np.int32)
        pr = R.Prompt(len(pt), np_ptr(pt, C.c_int32), len(hp), np_ptr(hp, C.c_int64), np_ptr(ht, C.c_int32), len(ci),
                      np_ptr(ci, C.c_int64), np_ptr(cl, C.c_int32), np_ptr(ct, C.c_int32), len(tt), np_ptr(tt, C.c_int32))
        cap = len(pt) + len(ht) + int(cl.sum()) + len(tt)
        tok = np.zeros(cap, np.int32); cls = np.zeros(cap, np.uint8); sid = np.zeros(cap, np.int64)
        soff = np.zeros(cap, np.int32); seg = np.zeros(3 + len(ci), np.int32)
        n = C.c_int32()
        check(lib().rc_decompose_prompt(C.byref(pr), cap, C.byref(n), np_ptr(tok, C.c_int32), np_ptr(cls, C.c_uint8),
                                        np_ptr(sid, C.c_int64), np_ptr(soff, C.c_int32), np_ptr(seg, C.c_int32)))
        idtok = np.array([int(t[0]) for t in cand_tokens], np.int32)
        return dict(tokens=tok[:n.value], cls=cls[:n.value], src_id=sid[:n.value], src_off=soff[:n.value],
                    seg_start=seg, cand_idtok=idtok)

    def assemble(self, layouts, prefix_id=0, miss_policy=R.RC_MISS_RECOMPUTE, gather_from=1, stream=None):
        """layouts: dicts with tokens, cls, src_id, src_off, cand_idtok (host arrays)."""
        n = len(layouts)
        reqs = (R.Request * n)()
        keep = []
        for i, lay in enumerate(layouts):
            arrs = [np.ascontiguousarray(lay["tokens"], np.int32), np.ascontiguousarray(lay["cls"], np.uint8),
                    np.ascontiguousarray(lay["src_id"], np.int64), np.ascontiguousarray(lay["src_off"], np.int32),
                    np.ascontiguousarray(lay["cand_idtok"], np.int32)]
            keep.append(arrs)
            hp = lay.get("hist_proto_dev")  # optional CUDA int32 tensor (NEXT-3 device-fed prototypes)
            reqs[i] = R.Request(len(arrs[0]), np_ptr(arrs[0], C.c_int32), np_ptr(arrs[1], C.c_uint8),
                                np_ptr(arrs[2], C.c_int64), np_ptr(arrs[3], C.c_int32), prefix_id, len(arrs[4]),
                                np_ptr(arrs[4], C.c_int32), hp.data_ptr() if hp is not None else None)
        seqs = np.zeros(n, np.uint64)
        missing = np.zeros(4096, np.uint64)
        nm = C.c_int32(len(missing))
        code = lib().rc_assemble(self.ctx, n, reqs, miss_policy, gather_from, np_ptr(seqs, C.c_uint64),
                                 np_ptr(missing, C.c_uint64), C.byref(nm), _stream(stream))
        self.last_missing = missing[:min(nm.value, len(missing))].copy()
        check(code)
        return seqs

    def _params(self, r_rev_bp, r_item_bp, check_layer, window, forced_sel, lam=1.0, attn_kernel=0, deterministic=0,
                gradual=0, r_start_rev_bp=None, r_start_item_bp=None):
        prm = R.PrefillParams(r_rev_bp, r_item_bp, lam, check_layer, window, None, None, attn_kernel, None,
                              int(deterministic), int(gradual),
                              int(r_rev_bp if r_start_rev_bp is None else r_start_rev_bp),
                              int(r_item_bp if r_start_item_bp is None else r_start_item_bp), None)
        keep = None
        if forced_sel is not None:
            off = np.zeros(len(forced_sel) + 1, np.int32)
            off[1:] = np.cumsum([len(s) for s in forced_sel])
            flat = np.ascontiguousarray(np.concatenate([np.asarray(s, np.int32) for s in forced_sel]), np.int32)
            prm.forced_sel = np_ptr(flat, C.c_int32)
            prm.forced_sel_off = np_ptr(off, C.c_int32)
            keep = (flat, off)
        return prm, keep

    def sel_count(self, seqs, r_rev_bp, r_item_bp, check_layer=1, window=0):
        seqs = np.ascontiguousarray(seqs, np.uint64)
        prm, _ = self._params(r_rev_bp, r_item_bp, check_layer, window, None)
        out = np.zeros(len(seqs), np.int32)
        check(lib().rc_sel_count(self.ctx, len(seqs), np_ptr(seqs, C.c_uint64), C.byref(prm), np_ptr(out, C.c_int32)))
        return out

    def selective_prefill(self, seqs, r_rev_bp, r_item_bp, check_layer=1, window=0, forced_sel=None, lam=1.0,
                          logits=True, cand_scores=True, sel_pos=True, hidden=False, n_cand=None, out=None,
                          stream=None, attn_kernel=0, score_out=None, deterministic=False, gradual=0,
                          r_start_rev_bp=None, r_start_item_bp=None, sel_trace=False):
        """Returns dict of CUDA tensors (logits, cand_scores, sel_pos, hidden) as requested. `out`
        may hold preallocated tensors with the same keys (reused; no allocation). score_out: optional
        int64 CUDA tensor [sum |U|] receiving the selection score of every U row (lam < 1: Eq. 3
        with the attention-mass term, NEXT-1). gradual > 0: gradual filtering from the r_start
        ratios at the check layer down to r at layer c + gradual (reading R-GF); sel_trace=True
        adds "sel_trace" (the positions of Sel_0 .. Sel_g, step-major) and "trace_off" (per step
        and request, offsets into it)."""
        seqs = np.ascontiguousarray(seqs, np.uint64)
        prm, keep = self._params(r_rev_bp, r_item_bp, check_layer, window, forced_sel, lam, attn_kernel, deterministic,
                                 gradual, r_start_rev_bp, r_start_item_bp)
        if score_out is not None:
            prm.score_out = score_out.data_ptr()
        res = dict(out) if out else {}
        if sel_trace and "sel_trace" not in res:
            rh0 = r_rev_bp if r_start_rev_bp is None else r_start_rev_bp
            ri0 = r_item_bp if r_start_item_bp is None else r_start_item_bp
            sizes = []
            for i in range(int(gradual) + 1):   # rc.h: r_i = r_start - floor((r_start - r) i / g)
                rh = rh0 - (rh0 - r_rev_bp) * i // gradual if gradual else r_rev_bp
                ri = ri0 - (ri0 - r_item_bp) * i // gradual if gradual else r_item_bp
                sizes.append(self.sel_count(seqs, rh, ri, check_layer, window))
            sizes = np.stack(sizes)
            res["trace_off"] = np.concatenate([[0], np.cumsum(sizes.ravel())]).astype(np.int64)
            res["sel_trace"] = torch.empty((int(sizes.sum()),), dtype=torch.int32, device=torch.device("cuda", self.device))
        if "sel_trace" in res:
            prm.sel_trace = res["sel_trace"].data_ptr()
        dev = torch.device("cuda", self.device)
        if (sel_pos or hidden) and ("sel_pos" not in res and "hidden" not in res):
            cnt = self.sel_count(seqs, r_rev_bp, r_item_bp, check_layer, window)
            S = int(cnt.sum())
            res["sel_off"] = np.concatenate([[0], np.cumsum(cnt)]).astype(np.int64)
        if logits and "logits" not in res:
            res["logits"] = torch.empty((len(seqs), self.shape.vocab), dtype=torch.float32, device=dev)
        if cand_scores and "cand_scores" not in res:
            res["cand_scores"] = torch.empty((int(n_cand),), dtype=torch.float32, device=dev)
        if sel_pos and "sel_pos" not in res:
            res["sel_pos"] = torch.empty((S,), dtype=torch.int32, device=dev)
        if hidden and "hidden" not in res:
            res["hidden"] = torch.empty((S, self.shape.d_model), dtype=torch.float32, device=dev)
        check(lib().rc_selective_prefill(self.ctx, len(seqs), np_ptr(seqs, C.c_uint64), C.byref(prm),
                                         _dptr(res.get("logits") if logits else None),
                                         _dptr(res.get("cand_scores") if cand_scores else None),
                                         _dptr(res.get("sel_pos") if sel_pos else None),
                                         _dptr(res.get("hidden") if hidden else None), _stream(stream)))
        return res

    def read_kv(self, seq, layer, n, stream=None):
        s = self.shape
        dev = torch.device("cuda", self.device)
        k = torch.empty((n, s.n_kv_heads, s.head_dim), dtype=torch.int16, device=dev)
        v = torch.empty_like(k)
        check(lib().rc_seq_read_kv(self.ctx, int(seq), layer, _dptr(k), _dptr(v), _stream(stream)))
        return k, v

    def export_kv(self, seq, pos0, n_tok, int8=False, stream=None):
        """rc_seq_export_kv: positions pos0.. of a sequence -> registration layout [n][L][2][Hk][dh]
        (bf16, or int8 codes + fp32 scales [n][L][2][Hk] per R15)."""
        s = self.shape
        dev = torch.device("cuda", self.device)
        shp = (n_tok, s.n_layers, 2, s.n_kv_heads, s.head_dim)
        kv = torch.empty(shp, dtype=torch.int8 if int8 else torch.bfloat16, device=dev)
        sc = torch.empty(shp[:4], dtype=torch.float32, device=dev) if int8 else None
        check(lib().rc_seq_export_kv(self.ctx, int(seq), int(pos0), int(n_tok), 1 if int8 else 0, _dptr(kv),
                                     _dptr(sc) if sc is not None else None, _stream(stream)))
        return (kv, sc) if int8 else kv

    def release(self, seqs):
        seqs = np.ascontiguousarray(seqs, np.uint64)
        lib().rc_release(self.ctx, len(seqs), np_ptr(seqs, C.c_uint64))

    def device_error_count(self):
        return int(lib().rc_device_error_count(self.ctx))

    def launch_count(self):
        return int(lib().rc_launch_count(self.ctx))

    def profile_begin(self):
        check(lib().rc_profile_begin(self.ctx))

    def profile_end(self):
        """-> {kind: dict(ms, launches, flops, bytes)} summed over the profiled launches."""
        n = len(R.KINDS)
        ms = (C.c_double * n)(); cnt = (C.c_int64 * n)(); fl = (C.c_double * n)(); by = (C.c_double * n)()
        check(lib().rc_profile_end(self.ctx, n, ms, cnt, fl, by))
        return {k: dict(ms=ms[i], launches=cnt[i], flops=fl[i], bytes=by[i]) for i, k in enumerate(R.KINDS)}

    # ------------------------------------------------------------------ multi-GPU
    def pool_export(self):
        h = (C.c_uint8 * 64)()
        rows = C.c_int64()
        check(lib().rc_pool_export(self.ctx, C.cast(h, C.c_void_p), C.byref(rows)))
        return bytes(h), rows.value

    def peer_attach(self, ranks, devices, handles, rows):
        n = len(ranks)
        r = np.ascontiguousarray(ranks, np.int32)
        d = np.ascontiguousarray(devices, np.int32)
        bufs = [(C.c_uint8 * 64).from_buffer_copy(h) for h in handles]
        hp = (C.c_void_p * n)(*[C.addressof(b) for b in bufs])
        rw = np.ascontiguousarray(rows, np.int64)
        check(lib().rc_peer_attach(self.ctx, n, np_ptr(r, C.c_int32), np_ptr(d, C.c_int32), C.cast(hp, R.PP),
                                   np_ptr(rw, C.c_int64)))

    def pool_list(self):
        """rc_pool_list: this pool's own item blocks -> (ids, rows, n_tokens, canon_pos)."""
        n = C.c_int32()
        lib().rc_pool_list(self.ctx, 0, None, None, None, None, C.byref(n))
        ids = np.zeros(n.value, np.uint64)
        rows = np.zeros(n.value, np.int64)
        nt = np.zeros(n.value, np.int32)
        cp = np.zeros(n.value, np.int32)
        check(lib().rc_pool_list(self.ctx, n.value, np_ptr(ids, C.c_uint64), np_ptr(rows, C.c_int64),
                                 np_ptr(nt, C.c_int32), np_ptr(cp, C.c_int32), C.byref(n)))
        return ids, rows, nt, cp

    def peer_directory(self, peer_rank, ids, rows, n_tokens, canon_pos):
        """rc_peer_directory: load an attached peer's item directory (from its pool_list)."""
        ids = np.ascontiguousarray(ids, np.uint64)
        rows = np.ascontiguousarray(rows, np.int64)
        nt = np.ascontiguousarray(n_tokens, np.int32)
        cp = np.ascontiguousarray(canon_pos, np.int32)
        check(lib().rc_peer_directory(self.ctx, int(peer_rank), len(ids), np_ptr(ids, C.c_uint64),
                                      np_ptr(rows, C.c_int64), np_ptr(nt, C.c_int32), np_ptr(cp, C.c_int32)))

    def fetch_remote(self, item_ids, owner_rank, stream=None):
        """rc_fetch_remote: pull item blocks from their owners' pools (one batched NVLink copy)."""
        ids = np.ascontiguousarray(item_ids, np.uint64)
        o = np.ascontiguousarray(owner_rank, np.int32)
        check(lib().rc_fetch_remote(self.ctx, len(ids), np_ptr(ids, C.c_uint64), np_ptr(o, C.c_int32),
                                    _stream(stream)))

    def fetch_host(self, item_ids, stream=None):
        """rc_fetch_host: host-tier item blocks -> the HBM remote-cache region on the copy engines."""
        ids = np.ascontiguousarray(item_ids, np.uint64)
        check(lib().rc_fetch_host(self.ctx, len(ids), np_ptr(ids, C.c_uint64), _stream(stream)))


    def semlib_build(self, proto_token, proto_offset, n_buckets, hyperplanes, seed):
        """rc_semlib_build (NEXT-3): host arrays; hyperplanes float32 [128][64]."""
        tok = np.ascontiguousarray(proto_token, np.int32)
        off = np.ascontiguousarray(proto_offset, np.int32)
        H = np.ascontiguousarray(hyperplanes, np.float32)
        check(lib().rc_semlib_build(self.ctx, len(tok), np_ptr(tok, C.c_int32), np_ptr(off, C.c_int32), int(n_buckets),
                                    np_ptr(H, C.c_float), int(seed)))

    def semlib_match(self, token, offset, stream=None):
        """rc_semlib_match: CUDA int32 tensors -> (proto ids int32, cosines float32) CUDA tensors."""
        n = token.numel()
        dev = torch.device("cuda", self.device)
        pid = torch.empty(n, dtype=torch.int32, device=dev)
        cos = torch.empty(n, dtype=torch.float32, device=dev)
        check(lib().rc_semlib_match(self.ctx, n, _dptr(token), _dptr(offset), _dptr(pid), _dptr(cos), _stream(stream)))
        return pid, cos


def diag_gemm(A, B, bn=256, stream=None):
    M, K = A.shape
    N = B.shape[0]
    Cm = torch.empty((M, N), dtype=torch.float32, device=A.device)
    check(lib().rc_diag_gemm(M, N, K, _dptr(A), _dptr(B), _dptr(Cm), bn, _stream(stream)))
    return Cm


def diag_gemm_add(A, B, X, transposed=False, stream=None):
    """X f32 [M][N] += A [M][K] B[N][K]^T in place (the residual-epilogue GEMM on its own)."""
    M, K = A.shape
    N = B.shape[0]
    check(lib().rc_diag_gemm_add(M, N, K, _dptr(A), _dptr(B), _dptr(X), 1 if transposed else 0, _stream(stream)))
    return X


def diag_deviation_select(k_new, k_st, v_new, v_st, cls, prefix_len, r_rev_bp, r_item_bp, window=0, stream=None):
    """bf16 (int16-viewed) CUDA tensors [n_u][width] -> (D uint64 numpy, Sel positions numpy)."""
    n_u, width = k_new.shape
    dev = torch.empty((n_u,), dtype=torch.int64, device=k_new.device)
    sel = torch.empty((n_u + 1,), dtype=torch.int32, device=k_new.device)
    cls = np.ascontiguousarray(cls, np.uint8)
    ns = C.c_int32()
    check(lib().rc_diag_deviation_select(n_u, width, _dptr(k_new), _dptr(k_st), _dptr(v_new), _dptr(v_st),
                                         np_ptr(cls, C.c_uint8), prefix_len, r_rev_bp, r_item_bp, window, _dptr(dev),
                                         _dptr(sel), C.byref(ns), _stream(stream)))
    return dev.cpu().numpy().view(np.uint64), sel[:ns.value].cpu().numpy()
