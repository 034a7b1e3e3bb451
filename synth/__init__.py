"""Seeded synthetic input generators (no method arithmetic). See synth/gen.py."""
from . import gen  # noqa: F401
