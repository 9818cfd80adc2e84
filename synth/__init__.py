"""Seeded synthetic input generators shared by tests, bench and oracle checks.

Holds NONE of the method's arithmetic (no returns, no priorities, no tree, no
gather logic): only random inputs with the shapes and value distributions of
the paper's workloads.
"""
from .workloads import *  # noqa: F401,F403
