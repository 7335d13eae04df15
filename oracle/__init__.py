"""Oracle for arXiv 2110.13638 (EDLaaS) -- TEST INFRASTRUCTURE ONLY.

A plain, slow, obviously-correct CPU implementation of what the GPU hot path
computes: Alg. 8 parameters, textbook RNS-CKKS (encode, Philox sampling, keygen,
encrypt/decrypt, add, scalar mul, tensor + key-switch, rescale) and the paper's
layer nodes (cross-correlation, sigma_a, dense).  Only tests/, __graft_entry__.smoke()
and bench.py's cpu_baseline / --impl reference legs may import it; the product path
(paper_2110_13638_b200/) never does and shares no code with it.

Parity status: every function here is pinned by tests/test_oracle_*.py against
something other than itself (O(N^2) definitions, schoolbook products, big-integer
CRT identities, closed forms, curand's Philox, float64 networks) -- see DESIGN.md.
"""
