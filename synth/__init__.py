"""Seeded synthetic input generators (no method arithmetic); see synth/matrices.py."""
from .matrices import *  # noqa: F401,F403
