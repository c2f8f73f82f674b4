"""CPU-side checks of the C-ABI library: it builds for sm_100a, loads, exports every symbol that
include/usk.h declares, and the binding refuses to run without it (no fallback)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "usk.h")


def _declared():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"USK_API\s+[\w\s\*]+?\b(usk_\w+)\s*\(", src)))


@pytest.fixture(scope="module")
def libpath():
    from paper_2506_17255_b200 import build as b
    return b.build()


def test_header_declares_boundary():
    names = _declared()
    for required in ("usk_plan_allocation", "usk_build", "usk_reconstruct", "usk_linear"):
        assert required in names
    assert len(names) >= 14


def test_library_exports_every_declared_symbol(libpath):
    lib = ctypes.CDLL(libpath)
    for name in _declared():
        assert hasattr(lib, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", libpath], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (usk_\w+)", out))
    assert set(_declared()) <= exported


def test_sm100a_code_in_library(libpath):
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", libpath], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_status_strings_and_host_errors(libpath):
    from paper_2506_17255_b200 import usk
    assert usk.lib.usk_status_string(3) == b"USK_EBUDGET"
    # argument validation happens before any device work
    with pytest.raises(usk.UskError) as e:
        usk.plan_allocation([(64, 64)], bpw=0.0)
    assert e.value.status == usk.EINVAL
    with pytest.raises(usk.UskError) as e:
        usk.plan_allocation([(64, 64)], bpw=1.0, rows=9)
    assert e.value.status == usk.EINVAL
    with pytest.raises(usk.UskError) as e:
        usk.plan_allocation([(0, 64)], bpw=1.0)
    assert e.value.status == usk.ESHAPE
    with pytest.raises(usk.UskError) as e:
        usk.plan_allocation([(64, 30)], bpw=1.0, dims_per_unit=4)
    assert e.value.status == usk.EINVAL


def test_binding_fails_loudly_without_library(tmp_path):
    code = ("import sys, types; sys.path.insert(0, %r);\n"
            "import paper_2506_17255_b200.usk as u\n") % ROOT
    env = dict(os.environ)
    # point the binding at a directory without the library
    fake = tmp_path / "paper_2506_17255_b200"
    fake.mkdir()
    (fake / "__init__.py").write_text("")
    (fake / "usk.py").write_text(open(os.path.join(ROOT, "paper_2506_17255_b200", "usk.py")).read())
    r = subprocess.run(["python", "-c", "import sys; sys.path.insert(0, %r); import paper_2506_17255_b200.usk"
                        % str(tmp_path)], capture_output=True, text=True, env=env)
    assert r.returncode != 0 and "libusk.so is missing" in r.stderr
