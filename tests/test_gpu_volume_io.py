"""GPU .vol IO: files written by the reference-format host
writer read straight into HBM (fp64 bit-exact, fp32 rounded), device writes
read back bit-exactly by the host reader, and the reference's format errors
(volumes.py:96-113) raise VolumeFormatError — also for a non-finite payload
detected on the device. Sizes cover several 32 MiB staging chunks."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2009_05473_b200 as pkg
    return pkg


@pytest.mark.parametrize("dims", [(3, 4, 5), (160, 128, 96)])
def test_volume_roundtrip_device(P, tmp_path, dims):
    import torch
    from paper_2009_05473_b200 import volumes as V
    rng = np.random.default_rng(sum(dims))
    v = P.Volume(rng.standard_normal(dims))
    f = tmp_path / "a.vol"
    P.write_volume(v, f)
    d64 = V.read_volume_device(f, precision="f64")
    assert d64.dtype == torch.float64 and np.array_equal(d64.cpu().numpy(), v.data)
    d32 = V.read_volume_device(f, precision="f32")
    assert np.array_equal(d32.cpu().numpy(), v.data.astype(np.float32))
    g = tmp_path / "b.vol"
    V.write_volume_device(d64, g)
    assert g.read_bytes() == f.read_bytes()
    V.write_volume_device(d32, g)
    assert np.array_equal(P.read_volume(g).data, v.data.astype(np.float32).astype(np.float64))


def test_volume_format_errors_device(P, tmp_path):
    from paper_2009_05473_b200 import volumes as V
    f = tmp_path / "a.vol"
    P.write_volume(P.Volume(np.ones((4, 4, 4))), f)
    raw = bytearray(f.read_bytes())
    bad = tmp_path / "bad.vol"
    for blob in (bytes(raw[:10]), b"XXXXXXXX" + bytes(raw[8:]), bytes(raw[:-8])):
        bad.write_bytes(blob)
        with pytest.raises(V.VolumeFormatError):
            V.read_volume_device(bad)
    nan = bytearray(raw)
    nan[20 + 8 * 5:20 + 8 * 6] = np.array([np.nan]).tobytes()
    bad.write_bytes(bytes(nan))
    with pytest.raises(V.VolumeFormatError):
        V.read_volume_device(bad)
