"""Seeded synthetic input generators shared by the oracle tests and the CUDA path.

This package holds no arithmetic of the method (§III): it only draws weights,
token ids, catalog/prototype structure, requests and pool bytes from fixed seeds.
"""
from .shapes import ModelShape, Workload, SHAPES, WORKLOADS, TINY, TINY_Q7, LLAMA3_8B, QWEN2_7B
from .shapes import CFG1, CFG1_Q7, CFG2, CFG3, CFG5, CFG5_2560, CFG5_4096, MIXED, MINI_L, MINI_Q, MINI_LLAMA, MINI_QWEN
from . import weights
from .weights import gen_weights, gen_tensor, subseed
from .workload import gen_catalog, gen_protos, gen_system_prompt, gen_request, gen_requests, proto_corpus, gen_mixed_requests
from . import pools
