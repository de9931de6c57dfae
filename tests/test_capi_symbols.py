"""The C-ABI library loads and exports every symbol include/sgs.h declares (no compute calls)."""
import ctypes
import os
import re

import paper_2504_15930_b200 as sgs
from paper_2504_15930_b200 import sgs as binding

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    src = open(os.path.join(ROOT, "include", "sgs.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(sgs_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    L = sgs.lib()
    names = declared_functions()
    assert len(names) >= 25
    for n in names:
        assert hasattr(L, n), n
    assert sorted(binding.EXPORTS) == names


def test_library_is_sm100a_native():
    # the fatbin carries sm_100a SASS with tcgen05 MMA and TMA (cuobjdump works without a GPU)
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", binding.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "UTCHMMA" in out and "UTMALDG" in out and "UBLKCP" in out and "LDTM" in out
    assert "sm_100a" in subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-lelf", binding.LIB_PATH],
                                       capture_output=True, text=True).stdout
