"""TEST INFRASTRUCTURE ONLY: CPU oracle for the DCT-domain block filter.

Two checkers, both loaded with ctypes:
  * ``Oracle``   - liboracle.so, the plain-C restatement (dctf_oracle.c);
  * ``Reference``- _ref/libdctf_ref.so, the unmodified reference headers
                   compiled in place (ref_harness.cc).
Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg may
import this package. The product package never does.
"""
from .oracle import LAPLACIAN3, MOTION_1x9, Gen, Oracle, Reference, reference_available  # noqa: F401
