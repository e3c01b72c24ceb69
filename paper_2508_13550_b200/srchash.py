"""Fingerprint of the evaluation kernels' sources.

An ncu capture's executed-flop-per-pair figure only describes the build it was taken
from; tools/ncu_eval_summary.py stores this hash in the profile and bench.py refuses a
profile whose hash differs from the sources it runs (the GPU box has no .git, so the
sources themselves are hashed, not a commit id).
"""
from __future__ import annotations

import hashlib
import os

_CSRC = os.path.join(os.path.dirname(os.path.abspath(__file__)), "csrc")
EVAL_KERNEL_SOURCES = ("interact.cu", "kernels_dev.cuh", "fastmath.cuh", "common.cuh", "log_table.inc")


def eval_kernel_sha256() -> str:
    h = hashlib.sha256()
    for name in EVAL_KERNEL_SOURCES:
        with open(os.path.join(_CSRC, name), "rb") as f:
            h.update(name.encode() + b"\0" + f.read())
    return h.hexdigest()
