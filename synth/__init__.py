"""Seeded synthetic inputs shared by the oracle (tests) and the product path.

Holds input formats and generators only -- none of the method's arithmetic
(see synth/format.py header).
"""
from . import format, abox, hyps  # noqa: F401
