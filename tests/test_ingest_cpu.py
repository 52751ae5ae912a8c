"""Recorded-stack ingest vs files written by the reference's own writers
(tests/golden/files: write_stack_raw / write_stack_tiff, ss/source.py:377-395)."""

import json
import os
import shutil

import numpy as np
import pytest

from paper_2211_00645_b200.errors import MetadataError
from paper_2211_00645_b200.ingest import load_stack, read_sidecar
from ssb_testutil import GOLDEN

FILES = os.path.join(GOLDEN, "files")


@pytest.mark.parametrize("name", ["stack.raw", "stack.tif"])
def test_reads_reference_files(name):
    stack, geom, timing = load_stack(os.path.join(FILES, name), pinned=False)
    want = np.load(os.path.join(FILES, "frames.npy"))
    np.testing.assert_array_equal(stack, want)
    # the reference's own replay of the raw file yields the same frames (ss/source.py:398-428)
    np.testing.assert_array_equal(stack, np.load(os.path.join(FILES, "replayed.npy")))
    assert (geom.slice_count, geom.frame_height_px, geom.frame_width_px) == (6, 10, 24)
    assert "exposure_ms" in timing


def test_sidecar_errors(tmp_path):
    raw = tmp_path / "s.raw"
    shutil.copy(os.path.join(FILES, "stack.raw"), raw)
    with pytest.raises(MetadataError, match="no sidecar"):
        load_stack(raw, pinned=False)
    side = json.load(open(os.path.join(FILES, "stack.json")))
    del side["geometry"]["alpha_deg"]
    json.dump(side, open(tmp_path / "s.json", "w"))
    with pytest.raises(MetadataError, match="geometry.alpha_deg"):
        read_sidecar(raw)
    side = json.load(open(os.path.join(FILES, "stack.json")))
    side["frames"] = 7
    json.dump(side, open(tmp_path / "s.json", "w"))
    with pytest.raises(MetadataError, match="sidecar says 7"):
        load_stack(raw, pinned=False)
    with open(tmp_path / "s.json", "w") as fh:
        fh.write("{not json")
    with pytest.raises(MetadataError, match="not valid JSON"):
        read_sidecar(raw)


def test_truncated_raw_rejected(tmp_path):
    raw = tmp_path / "t.raw"
    data = open(os.path.join(FILES, "stack.raw"), "rb").read()
    raw.write_bytes(data[:-2])
    shutil.copy(os.path.join(FILES, "stack.json"), tmp_path / "t.json")
    with pytest.raises(MetadataError, match="not a multiple"):
        load_stack(raw, pinned=False)


@pytest.mark.parametrize("name", ["stack.raw", "stack.tif"])
def test_reads_into_a_caller_buffer(name):
    want = np.load(os.path.join(FILES, "frames.npy"))
    buf = np.full(want.shape, 7, dtype=np.uint16)
    stack, _, _ = load_stack(os.path.join(FILES, name), out=buf)
    assert stack is buf
    np.testing.assert_array_equal(buf, want)
    with pytest.raises(MetadataError, match="out buffer"):
        load_stack(os.path.join(FILES, name), out=np.zeros((5, 10, 24), np.uint16))


def test_parallel_raw_read_in_small_pieces(tmp_path):
    # many pieces and a ragged last piece go to the right offsets
    from paper_2211_00645_b200.ingest import _read_parallel

    data = np.random.default_rng(3).integers(0, 256, 1_000_003, dtype=np.uint8)
    path = tmp_path / "blob.bin"
    data.tofile(path)
    out = np.zeros_like(data)
    _read_parallel(str(path), memoryview(out), data.size, threads=4, piece=4099)
    np.testing.assert_array_equal(out, data)
