"""Model shapes and workload configurations (SURVEY.md §8 "Model and prompt shapes").

Pure data: no arithmetic of the method lives here. Both the oracle (tests) and the
CUDA path (bench, tests) read these so that they run on identical inputs.
"""
from dataclasses import dataclass, field


@dataclass(frozen=True)
class ModelShape:
    name: str
    n_layers: int
    d_model: int
    n_heads: int
    n_kv_heads: int
    head_dim: int
    d_ff: int
    vocab: int
    rope_theta: float
    rms_eps: float
    qkv_bias: bool

    @property
    def group(self) -> int:
        return self.n_heads // self.n_kv_heads

    @property
    def q_dim(self) -> int:
        return self.n_heads * self.head_dim

    @property
    def kv_dim(self) -> int:
        return self.n_kv_heads * self.head_dim

    @property
    def kv_bytes_per_token_bf16(self) -> int:
        return self.n_layers * 2 * self.kv_dim * 2


# tiny: BASELINE.json configs[0] gives d=64, 4 heads; the rest are builder choices.
TINY = ModelShape("tiny", 2, 64, 4, 2, 16, 256, 512, 1e4, 1e-5, False)
# tiny-q7: GQA group 7 + QKV bias (exercises the Qwen2 code paths at test size), SURVEY §8 notes.
TINY_Q7 = ModelShape("tiny-q7", 2, 112, 7, 1, 16, 256, 512, 1e6, 1e-6, True)
# Public model configs (not from PAPER.md): Llama-3-8B and Qwen2-7B shapes.
LLAMA3_8B = ModelShape("llama3-8b", 32, 4096, 32, 8, 128, 14336, 128256, 5e5, 1e-5, False)
QWEN2_7B = ModelShape("qwen2-7b", 28, 3584, 28, 4, 128, 18944, 152064, 1e6, 1e-6, True)

# mini test shapes with the real head geometry (d_h = 128, GQA 4 / GQA 7 + bias) so that the
# tcgen05 attention and multi-tile paths run at sizes the oracle finishes in seconds.
MINI_LLAMA = ModelShape("mini-llama", 3, 1024, 8, 2, 128, 2048, 4096, 5e5, 1e-5, False)
MINI_QWEN = ModelShape("mini-qwen", 3, 896, 7, 1, 128, 2048, 4096, 1e6, 1e-6, True)

SHAPES = {s.name: s for s in (TINY, TINY_Q7, LLAMA3_8B, QWEN2_7B, MINI_LLAMA, MINI_QWEN)}


@dataclass(frozen=True)
class Workload:
    """Prompt recipe of one BASELINE config."""
    name: str
    shape: ModelShape
    prefix_len: int          # fixed system prompt P (207 tokens)
    hist_len: int            # history tokens (int8 prototype pool)
    n_cand: int              # candidate items per request
    item_len: int            # tokens per item block
    tail_len: int            # per-request instruction tail (FORCED)
    n_items: int             # catalog size
    n_clusters: int          # latent co-occurrence clusters
    n_protos: int            # prototype library size
    batch: int
    r_bp: int = 1500         # recompute ratio in basis points (r = 15%)
    review_len: int = 80     # ~80-token reviews

    @property
    def n(self) -> int:
        return self.prefix_len + self.hist_len + self.n_cand * self.item_len + self.tail_len


CFG1 = Workload("cfg1-tiny", TINY, 8, 64, 4, 16, 8, 64, 16, 256, 1)
CFG1_Q7 = Workload("cfg1-tiny-q7", TINY_Q7, 8, 64, 4, 16, 8, 64, 16, 256, 1)
CFG2 = Workload("cfg2-llama-1k", LLAMA3_8B, 207, 1024, 20, 64, 49, 4096, 256, 100_000, 1)
CFG3 = Workload("cfg3-llama-4k", LLAMA3_8B, 207, 640, 50, 64, 49, 4096, 256, 100_000, 32)
CFG5 = Workload("cfg5-qwen-8k", QWEN2_7B, 207, 1536, 100, 64, 49, 8192, 256, 100_000, 1)

# config 5 mixed batch: 55 % 2560, 35 % 4096, 10 % 8192 tokens on the Qwen2 shape, one catalog
CFG5_2560 = Workload("cfg5-qwen-2560", QWEN2_7B, 207, 1024, 20, 64, 49, 8192, 256, 100_000, 1)
CFG5_4096 = Workload("cfg5-qwen-4096", QWEN2_7B, 207, 640, 50, 64, 49, 8192, 256, 100_000, 1)
MINI_L = Workload("mini-llama", MINI_LLAMA, 64, 160, 8, 32, 16, 256, 16, 2048, 2)
MINI_Q = Workload("mini-qwen", MINI_QWEN, 64, 160, 8, 32, 16, 256, 16, 2048, 2)

WORKLOADS = {w.name: w for w in (CFG1, CFG1_Q7, CFG2, CFG3, CFG5, CFG5_2560, CFG5_4096, MINI_L, MINI_Q)}
MIXED = {"cfg5-mixed": ((CFG5_2560, 0.55), (CFG5_4096, 0.35), (CFG5, 0.10))}

assert CFG1.n == 144 and CFG2.n == 2560 and CFG3.n == 4096 and CFG5.n == 8192
assert CFG5_2560.n == 2560 and CFG5_4096.n == 4096
