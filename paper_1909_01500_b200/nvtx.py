"""Optional NVTX ranges around every binding call (SURVEY.md §5 tracing).

Set RPL_NVTX=1 before importing the package: each public function of `ops` and each
public method of SumTree / GatherPlan is wrapped in a `torch.cuda.nvtx` range named
after the ABI entry, so an nsys / ncu timeline shows the replay steps by name.  Off by
default (no wrapper, no overhead).
"""
from __future__ import annotations

import functools
import os


def _wrap(fn, name):
    import torch

    @functools.wraps(fn)
    def inner(*a, **k):
        torch.cuda.nvtx.range_push(name)
        try:
            return fn(*a, **k)
        finally:
            torch.cuda.nvtx.range_pop()

    return inner


def install(ops_module):
    if os.environ.get("RPL_NVTX") != "1":
        return False
    for name in list(getattr(ops_module, "__all__", [])):
        obj = getattr(ops_module, name)
        if isinstance(obj, type):
            for attr, fn in list(vars(obj).items()):
                if callable(fn) and not attr.startswith("_"):
                    setattr(obj, attr, _wrap(fn, f"rpl.{name}.{attr}"))
        elif callable(obj):
            setattr(ops_module, name, _wrap(obj, f"rpl.{name}"))
    return True
