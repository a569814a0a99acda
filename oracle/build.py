"""ORACLE — TEST INFRASTRUCTURE ONLY.  Build recipe for the CPU checkers.

1. `oracle/liboracle.so`: the C restatement `oracle/cdp_oracle.c`
   (gcc -O2 -ffp-contract=off, pthreads).
2. `oracle/_ref/_kernels.*.so`: the reference's own native kernel, compiled
   from its source where it lies (`/root/reference/pkg/src/cyclicdp/training/
   _kernels.pyx`) with Cython + gcc -O3, exactly the reference's build flags
   (`pkg/setup.py:10-19`).  Only done when /root/reference exists (this
   container); the GPU box uses the prebuilt file that travels with the repo.
   Intermediate C goes to `oracle/build/`; nothing reference-derived is
   committed (both dirs are git-ignored).
"""

from __future__ import annotations

import os
import subprocess
import sys
import sysconfig

HERE = os.path.dirname(os.path.abspath(__file__))
REF_PYX = "/root/reference/pkg/src/cyclicdp/training/_kernels.pyx"
LIB = os.path.join(HERE, "liboracle.so")
REF_DIR = os.path.join(HERE, "_ref")


def ref_module_path() -> str:
    suffix = sysconfig.get_config_var("EXT_SUFFIX") or ".so"
    return os.path.join(REF_DIR, "_kernels" + suffix)


def build_oracle(force: bool = False) -> str:
    src = os.path.join(HERE, "cdp_oracle.c")
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(src):
        subprocess.check_call(
            ["gcc", "-O2", "-ffp-contract=off", "-fPIC", "-shared", "-pthread", src, "-o", LIB, "-lm"]
        )
    return LIB


def build_ref(force: bool = False):
    out = ref_module_path()
    if not os.path.exists(REF_PYX):
        return out if os.path.exists(out) else None
    if os.path.exists(out) and not force:
        return out
    os.makedirs(os.path.join(HERE, "build"), exist_ok=True)
    os.makedirs(REF_DIR, exist_ok=True)
    c_file = os.path.join(HERE, "build", "_kernels.c")
    subprocess.check_call(
        [sys.executable, "-m", "cython", "-3", "--module-name", "_kernels", REF_PYX, "-o", c_file]
    )
    import numpy as np

    inc = [sysconfig.get_paths()["include"], np.get_include()]
    cmd = ["gcc", "-O3", "-fPIC", "-shared", "-fwrapv", c_file, "-o", out, "-lm"]
    for d in inc:
        cmd.insert(1, f"-I{d}")
    subprocess.check_call(cmd)
    return out


def build(force: bool = False):
    build_oracle(force)
    build_ref(force)


if __name__ == "__main__":
    build(force="--force" in sys.argv)
    print(LIB, ref_module_path())
