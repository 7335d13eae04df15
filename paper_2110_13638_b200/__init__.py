"""B200-native hot path of arXiv 2110.13638 (EDLaaS): homomorphic inference of the
paper's node-centric network over RNS-CKKS, behind the C-ABI in include/edl.h.

Modules: ``edl`` (ctypes binding of libedl.so), ``graph`` (Alg. 1-5 firing engine),
``networks`` (C0/C1/C3 chains), ``build`` (nvcc build of libedl.so for sm_100a).
"""
