"""CPU: the C-ABI library loads and exports every symbol of include/*.h."""

from __future__ import annotations

import glob
import os
import re

from conftest import ROOT


def _declared():
    names = set()
    for h in glob.glob(os.path.join(ROOT, "include", "*.h")):
        text = open(h).read()
        names |= set(re.findall(r"\b(gp_[a-z_]+)\s*\(", text))
    return names


def test_library_exports_all_declared_symbols():
    from paper_2007_16076_b200 import _lib, build

    build.build()
    L = _lib.load_library(require_device=False)
    declared = _declared()
    assert declared >= {"gp_run", "gp_propagate", "gp_store_fill_tree"}
    missing = [s for s in declared if not hasattr(L, s)]
    assert not missing
    assert set(_lib.EXPORTS) == declared


def test_library_is_sm100a():
    import subprocess

    from paper_2007_16076_b200 import build

    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", build.OUT],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_error_message_without_device():
    from paper_2007_16076_b200 import _lib

    L = _lib.load_library(require_device=False)
    assert L.gp_version() >= 1
    assert isinstance(L.gp_last_error(), bytes)
