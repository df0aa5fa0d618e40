"""CPU parity oracle for the PacTrain gradient-sync hot path.

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's CPU-baseline / reference arm -- never by the product package
(paper_2505_18563_b200/), which fails loudly without its CUDA library.

Two backends, both plain ctypes over numpy arrays:

* ``port``: oracle/pact_oracle.c, the C restatement of the reference
  functions (each cites its reference file:line).
* ``ref``: oracle/_ref/libpactref.so, the reference's own sources compiled
  in place (namespace renamed to ``pactref``) plus oracle/ref_shim.cpp. It is
  used to pin ``port`` and to time the reference CPU path.
"""
from .oracle import (  # noqa: F401
    Port,
    Ref,
    build,
    port,
    ref,
    ref_available,
    words_from_bits,
    bits_from_words,
)
