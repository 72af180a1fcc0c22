"""Seeded synthetic inputs shared by oracle/ and the CUDA path (no method arithmetic)."""
from .circuits import *  # noqa
