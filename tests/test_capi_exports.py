"""The C-ABI library builds, loads without a GPU and exports every declared symbol.

No compute calls here (no GPU in the CPU suite); the product path must fail
loudly — a CUDA error, never a CPU fallback — when no device is present.
"""

import ctypes
import os
import re

import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "wos_b200.h")


def _declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(wos_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_abi():
    names = _declared()
    for must in ("wos_estimate", "wos_estimate_host", "wos_walk_rows", "wos_walk_rows_host",
                 "wos_philox4x64", "wos_check_interior", "wos_problem_set_create",
                 "wos_context_create", "wos_probe_peaks"):
        assert must in names


def test_library_exports_every_declared_symbol():
    from paper_2603_01193_b200 import _lib

    lib = ctypes.CDLL(_lib.lib_path)
    missing = [n for n in _declared() if not hasattr(lib, n)]
    assert not missing, missing


def test_python_binding_covers_the_header():
    from paper_2603_01193_b200 import _lib

    assert set(_declared()) == set(_lib.EXPORTED_SYMBOLS)


def test_abi_version_and_error_string():
    from paper_2603_01193_b200 import _lib

    L = _lib.load_library()
    assert L.wos_abi_version() == _lib.ABI_VERSION == 4
    assert isinstance(_lib.last_error(), str)


def test_library_is_built_for_sm_100a():
    import subprocess

    from paper_2603_01193_b200 import _lib

    out = subprocess.run(["cuobjdump", "--list-elf", _lib.lib_path], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_no_gpu_fails_loudly_not_silently():
    """Without a CUDA device the product path raises; it never computes on the CPU."""
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_2603_01193_b200 import BoxDomain, Problem, WalkConfig, _lib, estimate, specs

    prob = Problem(BoxDomain([0, 0], [1, 1]), boundary_spec=specs.const_boundary(0.0))
    with pytest.raises(_lib.WosError):
        estimate(prob, [[0.5, 0.5]], 4, WalkConfig())


def test_missing_library_raises(tmp_path):
    from paper_2603_01193_b200 import _lib

    with pytest.raises(_lib.WosUnavailableError):
        _lib.load_library(str(tmp_path / "nope.so"))


def test_ctypes_structs_match_the_c_header(tmp_path):
    """The ctypes mirrors of wos_problem / wos_walk_config (and the INTEGRATION.md stub,
    which uses the same fields) have the C header's size and field offsets."""
    import ctypes
    import os
    import shutil
    import subprocess

    from paper_2603_01193_b200 import _lib

    cc = shutil.which("gcc") or shutil.which("cc")
    if cc is None:  # pragma: no cover - the image has gcc
        import pytest

        pytest.skip("no C compiler")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    src = tmp_path / "layout.c"
    fields = {"wos_problem": [f for f, _ in _lib.WosProblem._fields_],
              "wos_walk_config": [f for f, _ in _lib.WosWalkConfig._fields_]}
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "wos_b200.h"', "int main(void) {"]
    for st, fs in fields.items():
        lines.append(f'  printf("{st} %zu\\n", sizeof({st}));')
        for f in fs:
            lines.append(f'  printf("{st}.{f} %zu\\n", offsetof({st}, {f}));')
    lines += ["  return 0;", "}"]
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.run([cc, "-I", os.path.join(root, "include"), str(src), "-o", str(exe)], check=True)
    got = dict(line.split() for line in subprocess.run([str(exe)], capture_output=True, text=True,
                                                       check=True).stdout.splitlines())
    for st, cls in (("wos_problem", _lib.WosProblem), ("wos_walk_config", _lib.WosWalkConfig)):
        assert int(got[st]) == ctypes.sizeof(cls), st
        for f in fields[st]:
            assert int(got[f"{st}.{f}"]) == getattr(cls, f).offset, (st, f)
