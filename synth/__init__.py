"""Seeded synthetic inputs (no method arithmetic); shared by oracle tests, GPU tests and bench."""
from .generators import *  # noqa: F401,F403
