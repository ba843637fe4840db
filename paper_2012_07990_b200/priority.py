"""Delta-stepping bucket queue constants (reference priority.py).

The two-bucket queue itself (current + far with lazy re-bucketing and stale
filtering, priority.py:17-118) lives on the device inside the SSSP driver
(csrc/sssp.cu); its observable behaviour is pinned by tests/test_sssp_*.
"""

UNREACHED = 2**64 - 1  # reserved infinity sentinel for 64-bit priorities (priority.py:14)
