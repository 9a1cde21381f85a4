"""Build the reference CPU implementation into ``oracle/_ref/`` (checker only).

TEST INFRASTRUCTURE. Nothing under ``oracle/`` is part of the product: only
``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s reference /
cpu_baseline legs may import it.

Recipe (does NOT run the reference's own build system, ``pkg/setup.py``):

1. copy the reference's pure-Python package sources
   ``/root/reference/pkg/src/pisoflow/*.py`` into ``oracle/_ref/pisoflow/``
   (git-ignored; it travels to the GPU box with the snapshot like any other
   built artefact, because ``/root/reference`` does not exist there);
2. translate the compiled kernel lane ``_kernels_c.pyx``
   (``S/_kernels_c.pyx:1-149``) to C with the ``cython`` compiler;
3. compile it with ``gcc -O3 -shared -fPIC`` against the Python and NumPy
   headers, exactly the flags ``pkg/setup.py:30-42`` asks for.

``python oracle/build_ref.py`` is idempotent; it is a no-op when
``/root/reference`` is absent (on the GPU box the prebuilt files are used).
Afterwards ``PYTHONPATH=oracle/_ref python -c 'import pisoflow.kernels as k;
print(k.LANE)'`` prints ``c``.
"""

import os
import shutil
import subprocess
import sys
import sysconfig

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SRC = "/root/reference/pkg/src/pisoflow"
OUT = os.path.join(HERE, "_ref", "pisoflow")


def _ext_suffix():
    return sysconfig.get_config_var("EXT_SUFFIX") or ".so"


def build(verbose=False):
    if not os.path.isdir(REF_SRC):
        return os.path.isdir(OUT)
    os.makedirs(OUT, exist_ok=True)
    for name in sorted(os.listdir(REF_SRC)):
        if name.endswith(".py"):
            src = os.path.join(REF_SRC, name)
            dst = os.path.join(OUT, name)
            if (not os.path.exists(dst)
                    or os.path.getmtime(dst) < os.path.getmtime(src)):
                shutil.copy2(src, dst)
    so = os.path.join(OUT, "_kernels_c" + _ext_suffix())
    pyx = os.path.join(REF_SRC, "_kernels_c.pyx")
    if os.path.exists(so) and os.path.getmtime(so) >= os.path.getmtime(pyx):
        return True
    import numpy as np
    c_file = os.path.join(HERE, "_ref", "_kernels_c.c")
    subprocess.run([sys.executable, "-m", "cython", "-3", "-o", c_file,
                    "--module-name", "pisoflow._kernels_c", pyx], check=True,
                   capture_output=not verbose)
    inc = [sysconfig.get_paths()["include"], np.get_include()]
    cmd = ["gcc", "-O3", "-shared", "-fPIC", "-o", so, c_file,
           "-DNPY_NO_DEPRECATED_API=NPY_1_7_API_VERSION"]
    cmd += [f"-I{p}" for p in inc]
    subprocess.run(cmd, check=True, capture_output=not verbose)
    return True


def ref_path():
    """Directory to put on sys.path to import the reference ``pisoflow``."""
    return os.path.join(HERE, "_ref")


if __name__ == "__main__":
    ok = build(verbose=True)
    print("oracle/_ref ready" if ok else "reference absent; nothing built")
