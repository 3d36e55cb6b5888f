"""CPU-side checks of the C-ABI library: it loads, exports every symbol the
header declares, and its host-only geometry helper agrees with the oracle.
No GPU work is issued here."""
import re
from pathlib import Path

import numpy as np
import pytest

import sfw3d_oracle as O
from paper_2009_05473_b200 import _native as N

ROOT = Path(__file__).resolve().parents[1]


def header_symbols():
    text = (ROOT / "include" / "sfw3d_cuda.h").read_text()
    return sorted(set(re.findall(r"\b(sfw3d_[a-z0-9_]+)\s*\(", text)))


def test_header_matches_binding_table():
    assert header_symbols() == sorted(N.EXPORTS)


def test_library_exports_every_header_symbol():
    lib = N.lib()
    for name in header_symbols():
        assert hasattr(lib, name), name
    assert lib.sfw3d_abi_version() == 3


def test_library_is_sm100a():
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", str(N.lib_path())], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_geometry_matches_oracle():
    rng = np.random.default_rng(1)
    for dims in ((64, 64, 64), (13, 16, 11), (128, 96, 40)):
        rows = np.column_stack([
            rng.uniform(0.1, 2, 200),
            rng.uniform(-3, dims[0] + 3, 200), rng.uniform(-3, dims[1] + 3, 200),
            rng.uniform(-3, dims[2] + 3, 200),
            rng.uniform(0.7, 3.2, 200), rng.uniform(1.1, 3.0, 200)])
        rows[:10, 1:4] = np.round(rows[:10, 1:4]) + 0.5   # half-even ties
        rows[10:20, 5] = 2.0
        radius, start, length, full = N.atom_geometry(dims, rows)
        for i, r in enumerate(rows):
            R = O.support_radius(r[4], r[5])
            assert radius[i] == R
            for a in range(3):
                idx, off = O.axis_box(dims[a], r[1 + a], R)
                assert length[i, a] == len(idx)
                if full[i, a]:
                    assert len(idx) == dims[a] and 2 * R + 1 >= dims[a]
                else:
                    assert start[i, a] == int(np.round(r[1 + a])) - R
                    assert idx[0] == start[i, a] % dims[a]


def test_geometry_rejects_bad_atoms():
    with pytest.raises(ValueError):
        N.atom_geometry((8, 8, 8), np.array([[1.0, 1, 1, 1, 0.0, 2.0]]))
    with pytest.raises(ValueError):
        N.atom_geometry((8, 8, 8), np.array([[1.0, 1, 1, np.nan, 1.0, 2.0]]))
    with pytest.raises(ValueError):
        N.atom_geometry((8, 0, 8), np.array([[1.0, 1, 1, 1, 1.0, 2.0]]))


def test_device_calls_fail_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(RuntimeError):
        N.context()


REFERENCE_SRC = Path("/root/reference/pkg/src")


@pytest.mark.skipif(not (REFERENCE_SRC / "sfw3d").exists(), reason="reference not present")
def test_integration_snippet_rebinds_real_reference():
    """INTEGRATION.md's binding, executed verbatim against the real sfw3d
    0.1.0 (build container only; no compute): every name the reference's
    modules bind by import is replaced in every namespace, incl. the CLI's
    solvers and the Psf class the CLI constructs (cli.py:20-23, 85-86)."""
    import subprocess
    import sys
    code = f"""
import sys
sys.path[:0] = [{str(REFERENCE_SRC)!r}, {str(ROOT)!r}, {str(ROOT / 'tests')!r}]
import sfw3d, sfw3d.cli, sfw3d.experiment
from integration_snippet import load_snippet
done = load_snippet()["enable"]("f64")
import paper_2009_05473_b200 as gpu
want = [("sfw3d.cli", "bsfw"), ("sfw3d.cli", "sfw"), ("sfw3d.forward", "Psf"),
        ("sfw3d.solvers", "certificate_max"), ("sfw3d.solvers", "local_descent"),
        ("sfw3d.certificate", "eta_field"), ("sfw3d.experiment", "forward"), ("sfw3d", "bsfw")]
for m, n in want:
    assert (m, n) in done, (m, n)
    assert getattr(sys.modules[m], n) is getattr(gpu, n), (m, n)
print("rebound", len(done))
"""
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    assert "rebound" in out.stdout
