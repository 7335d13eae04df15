"""Seeded synthetic inputs shared by the oracle tests and the GPU path.

Holds none of the method's arithmetic: only numpy PCG64 draws with the shapes and
value distributions of BASELINE.json's configs; see DESIGN.md
"Input recipe".
"""
from .inputs import *  # noqa: F401,F403
