"""Content hash of the native sources (csrc/ + include/), stamped into the
ncu summaries under profiles/ and checked by bench.py, so a committed
counter file is only quoted for the code it was captured on.  (The GPU box
gets a snapshot without .git, so this hashes file contents, not commits.)"""
from __future__ import annotations

import hashlib
import os

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)


def native_files():
    out = []
    for d, exts in ((os.path.join(HERE, "csrc"), (".cu", ".cuh", ".cpp", ".hpp", ".h")),
                    (os.path.join(REPO, "include"), (".h", ".hpp"))):
        for f in sorted(os.listdir(d)):
            if f.endswith(exts):
                out.append(os.path.join(d, f))
    return out


def csrc_sha256() -> str:
    h = hashlib.sha256()
    for p in native_files():
        h.update(os.path.relpath(p, REPO).encode())
        h.update(b"\0")
        with open(p, "rb") as f:
            h.update(f.read())
        h.update(b"\0")
    return h.hexdigest()
