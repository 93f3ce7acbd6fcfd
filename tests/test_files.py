"""Record / label file formats -- host-side, no GPU:
round trips in both layouts, the header checksum equals the reference's
dataset_checksum (Appendix A vectors), malformed files raise IoError, u8
labels reject classes >= 256."""
import os

import numpy as np
import pytest

import paper_1111_1373_b200 as st
from paper_1111_1373_b200.errors import ArgumentError, IoError


@pytest.mark.parametrize("layout", ["aos", "soa"])
def test_record_file_round_trip(tmp_path, layout):
    x = st.generate_synthetic_dataset(1000, 19, 2)
    p = str(tmp_path / f"d_{layout}.strec")
    st.save_dataset_bin(p, x, layout=layout)
    info = st.dataset_info(p)
    assert info["count"] == 1000 and info["arity"] == 19 and info["layout"] == layout
    assert info["checksum"] == st.dataset_checksum(x)
    assert os.path.getsize(p) == 64 + 1000 * 19 * 4
    d = st.load_dataset_bin(p, verify=True)
    assert np.array_equal(d.values(), x)
    part = st.load_dataset_bin(p, first=123, count=77)
    assert np.array_equal(part.values(), x[123:200])


def test_header_checksum_is_reference_dataset_checksum(tmp_path, co):
    # Appendix A: data(16384, 19, 2) tiled 4x -> 0x33d552cf6075468f
    x = np.tile(co.gen_dataset(16384, 19, 2), (4, 1))
    p = str(tmp_path / "paper.strec")
    st.save_dataset_bin(p, x)
    assert st.dataset_info(p)["checksum"] == 0x33d552cf6075468f


def test_empty_and_no_checksum(tmp_path):
    p = str(tmp_path / "e.strec")
    st.save_dataset_bin(p, np.zeros((0, 3), np.float32), checksum=False)
    assert st.dataset_info(p)["count"] == 0 and st.dataset_info(p)["checksum"] is None
    assert st.load_dataset_bin(p).count() == 0
    with pytest.raises(IoError):
        st.load_dataset_bin(p, verify=True)  # nothing to verify against


def test_malformed_record_files(tmp_path):
    x = st.generate_synthetic_dataset(10, 4, 1)
    p = str(tmp_path / "ok.strec")
    st.save_dataset_bin(p, x)
    raw = open(p, "rb").read()
    bad = tmp_path / "bad.strec"
    bad.write_bytes(b"NOTMAGIC" + raw[8:])
    with pytest.raises(IoError):
        st.dataset_info(str(bad))
    bad.write_bytes(raw[:-4])  # truncated
    with pytest.raises(IoError):
        st.load_dataset_bin(str(bad))
    flipped = bytearray(raw)
    flipped[64 + 5] ^= 0x01  # payload changed, header checksum stale
    bad.write_bytes(bytes(flipped))
    with pytest.raises(IoError, match="checksum"):
        st.load_dataset_bin(str(bad), verify=True)
    with pytest.raises(IoError):
        st.dataset_info(str(tmp_path / "missing.strec"))
    with pytest.raises(ArgumentError):
        st.load_dataset_bin(p, first=5, count=6)


@pytest.mark.parametrize("width", [1, 4])
def test_label_file_round_trip(tmp_path, width):
    lab = np.random.default_rng(3).integers(0, 200, 5000).astype(np.uint32)
    p = str(tmp_path / f"l{width}.stlab")
    st.save_labels_bin(p, lab, width)
    assert os.path.getsize(p) == 32 + 5000 * width
    assert np.array_equal(st.load_labels_bin(p), lab)


def test_u8_labels_reject_large_classes(tmp_path):
    with pytest.raises(ArgumentError):
        st.save_labels_bin(str(tmp_path / "x.stlab"), np.array([3, 256], np.uint32), 1)
    with pytest.raises(ArgumentError):
        st.save_labels_bin(str(tmp_path / "x.stlab"), np.array([3], np.uint32), 2)
