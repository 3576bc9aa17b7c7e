"""CPU checks of the offline pipeline's host side: the `.tnsc` reader/writer against a file
the reference itself wrote (sf/containers.py), and the seeded predictor init draws
(sf/predictor.py:194-206) against the reference's."""

import numpy as np
import pytest

from paper_2510_15964_b200 import tnsc
from tests.conftest import GOLDEN


def test_reads_reference_file(golden):
    g = golden("offline")
    t, col = tnsc.load_tensors(GOLDEN / "ref_container.tnsc")
    assert list(t) == list(g["ct/names"])
    assert col == {"colmaj"}
    for k in t:
        np.testing.assert_array_equal(t[k], g[f"ct/{k}"])
        assert t[k].dtype == g[f"ct/{k}"].dtype
    assert t["colmaj"].flags.f_contiguous


def test_writes_reference_bytes(golden, tmp_path):
    g = golden("offline")
    arrays = {str(k): g[f"ct/{k}"] for k in g["ct/names"]}
    tnsc.save_tensors(tmp_path / "x.tnsc", arrays, column_major={"colmaj"})
    assert (tmp_path / "x.tnsc").read_bytes() == (GOLDEN / "ref_container.tnsc").read_bytes()


def test_container_errors(tmp_path):
    with pytest.raises(tnsc.ContainerError):
        tnsc.save_tensors(tmp_path / "a.tnsc", {"x": np.zeros(3, np.int32)})
    with pytest.raises(tnsc.ContainerError):
        tnsc.save_tensors(tmp_path / "a.tnsc", {"x": np.zeros(3)}, column_major={"y"})
    (tmp_path / "bad.tnsc").write_bytes(b"NOPE" + bytes(20))
    with pytest.raises(tnsc.ContainerError):
        tnsc.load_tensors(tmp_path / "bad.tnsc")
    (tmp_path / "empty.tnsc").write_bytes(b"")
    with pytest.raises(tnsc.ContainerError):
        tnsc.load_tensors(tmp_path / "empty.tnsc")
    tnsc.save_tensors(tmp_path / "t.tnsc", {"x": np.arange(10.0)})
    data = (tmp_path / "t.tnsc").read_bytes()
    (tmp_path / "trunc.tnsc").write_bytes(data[:-8])
    with pytest.raises(tnsc.ContainerError):
        tnsc.load_tensors(tmp_path / "trunc.tnsc")
    (tmp_path / "ver.tnsc").write_bytes(data[:4] + (2).to_bytes(4, "little") + data[8:])
    with pytest.raises(tnsc.ContainerError):
        tnsc.load_tensors(tmp_path / "ver.tnsc")


def test_init_draws_match_reference(golden):
    from paper_2510_15964_b200 import offline as OF

    g = golden("offline")
    ap = OF.init_attn_predictor(48, 3, rank=None, seed=12)
    np.testing.assert_array_equal(np.stack(ap.wq_hat), g["init/wq"])
    np.testing.assert_array_equal(np.stack(ap.wk_hat), g["init/wk"])
    np.testing.assert_array_equal(OF.init_mlp_predictor(48, 5, seed=13).wa_hat, g["init/wa"])
