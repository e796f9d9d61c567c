"""Locate and import the genuine reference package -- TEST / BASELINE
INFRASTRUCTURE ONLY (tests/, __graft_entry__, bench.py's reference arm).

The reference (`seriesaug`, pure Python over numpy/scipy) lives read-only at
/root/reference/pkg in the build container.  `build()` installs it unmodified
into oracle/_ref/ (git-ignored, travels to the GPU box with the snapshot, like
a compiled reference would), so the reference's own `Pipeline.run` can be
timed and used as a checker where /root/reference does not exist.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
REF_TARGET = os.path.join(HERE, "_ref")
REF_SOURCE = "/root/reference/pkg"


def build() -> str | None:
    """Install the reference from its own sources into oracle/_ref (a copy of
    the source tree under /tmp is built, since the original is read-only).
    No-op when the reference is absent (GPU box) or already installed."""
    if os.path.isdir(os.path.join(REF_TARGET, "seriesaug")):
        return REF_TARGET
    if not os.path.isdir(REF_SOURCE):
        return None
    with tempfile.TemporaryDirectory() as tmp:
        src = os.path.join(tmp, "pkg")
        shutil.copytree(REF_SOURCE, src, ignore=shutil.ignore_patterns("frontend", "tests", "*.pyc"))
        r = subprocess.run([sys.executable, "-m", "pip", "install", "--quiet", "--no-index", "--no-deps",
                            "--no-build-isolation", "--target", REF_TARGET, src],
                           capture_output=True, text=True)
        if r.returncode != 0:
            # pure-Python package: the wheel build is a copy of src/seriesaug
            shutil.rmtree(REF_TARGET, ignore_errors=True)
            shutil.copytree(os.path.join(src, "src", "seriesaug"), os.path.join(REF_TARGET, "seriesaug"))
    return REF_TARGET


def location() -> str | None:
    if os.path.isdir(os.path.join(REF_TARGET, "seriesaug")):
        return REF_TARGET
    if os.path.isdir(os.path.join(REF_SOURCE, "src", "seriesaug")):
        return os.path.join(REF_SOURCE, "src")
    return None


def import_reference():
    """The reference's `seriesaug` module (oracle/_ref first)."""
    if "seriesaug" in sys.modules:
        return sys.modules["seriesaug"]
    loc = location()
    if loc is None:
        raise ImportError("the reference package is not installed (run __graft_entry__.build())")
    if loc not in sys.path:
        sys.path.insert(0, loc)
    import seriesaug

    return seriesaug
