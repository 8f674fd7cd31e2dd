"""CPU oracle of RcLLM's selective-attention prefill (arxiv 2605.07443, §III-C).

TEST INFRASTRUCTURE ONLY. Nothing in the product path (paper_2605_07443_b200/) may import,
call, link or execute anything under oracle/. Only tests/, __graft_entry__.smoke() and the
cpu_baseline / --impl reference legs of bench.py use it.

Plain, slow, obviously correct numpy: fp64 for the transformer arithmetic (the paper fixes
no precision), and the exact fp32 / integer operation sequences of SURVEY.md readings
R4 (fixed-point deviation), R6 (top-k order), R13 (RoPE tables and rotation) and R15
(int8 dequantisation) wherever a bit-exact result is defined. Shares no code with the
CUDA path; its inputs come from rcgen/ (seeded generators) only.

Modules
  numerics   bf16 RNE, RoPE tables / rotation, int8 dequant, fixed-point deviation
  layout     decompose_prompt / classify_tokens / budgets
  model      O-FULL: textbook Llama/Qwen2 prefill, Eq. 1
  assemble   O-ASM: gather + dequant + Delta-RoPE
  select     Eq. 3 importance score, heavy-hitter selection
  selective  O-SEL: selective recompute layer loop + readout

Parity unpinned: the fidelity of selective vs full prefill needs trained
weights and datasets; rel-L2(O-SEL, O-FULL) is only reported as a diagnostic.
"""
