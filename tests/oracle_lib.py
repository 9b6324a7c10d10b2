"""Test-side alias of oracle/pyoracle.py (the CPU numeric oracle bindings)."""
from oracle.pyoracle import *  # noqa: F401,F403
