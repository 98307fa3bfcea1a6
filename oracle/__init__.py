"""oracle/ -- TEST INFRASTRUCTURE ONLY.

A plain, slow, obviously-correct CPU implementation of what the Silenzio hot
path computes: TFHE keygen / encryption / decryption (numpy glue over plain C
loops), keyswitch, modulus switch, blind rotation with exact schoolbook
negacyclic products mod 2^64, sample extraction, the atomic-pattern PBS, and
the cleartext gadget reference (RNS, MRNS, Alg. 1-5).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
leg may import this package. It shares no code with paper_2504_17785_b200/
(the CUDA product path); both consume the seeded draws of synth/.

Parity status per function is listed in DESIGN.md §Oracle pins; a function with
no independent pin says "parity unpinned" in its docstring.
"""
from . import native  # noqa: F401
from .tfhe import *  # noqa: F401,F403
