"""`ising-model v1` documents: the product's reader/writer against the reference's
own (compiled unmodified into oracle/_ref) and against committed golden documents written by the
reference; parse errors carry the reference's 1-based line numbers and status codes
(ref: proj/src/model_io.cpp:45-226, proj/tests/test_model_io.cpp)."""
from pathlib import Path

import numpy as np
import pytest

import paper_1004_0024_b200 as ib
from paper_1004_0024_b200 import _lib, instances as ins
from helpers import product_model

GOLDEN = Path(__file__).resolve().parent / "golden"
KEYS = ("h", "offsets", "targets", "couplings", "tau_counts")


def sample_csrs():
    layered = ins.build_layered_csr(*ins.layered_spec(12, 7), 5, 1.5)
    generic = ins.cubic_mixed_degree(4, 21)
    tilted = ins.build_layered_csr(*ins.layered_spec(8, 3, h_sigma=0.0), 4, -0.375)
    tilted["h"][3] = np.float32(-0.0)  # a negative zero must survive the round trip
    return {"layered_12x5": layered, "generic_mixed": generic, "layered_8x4_zero_h": tilted}


def assert_same_csr(a, b):
    def column(csr, key):  # generic instances may leave tau_counts out: all zero
        value = csr.get(key)
        return np.zeros(len(csr["h"]), np.uint8) if value is None else np.ascontiguousarray(value)
    for key in KEYS:
        assert np.array_equal(column(a, key).view(np.uint8), column(b, key).view(np.uint8)), key


@pytest.mark.parametrize("name", ["layered_12x5", "generic_mixed", "layered_8x4_zero_h"])
def test_writer_matches_golden_documents_written_by_the_reference(lib, name):
    csr = sample_csrs()[name]
    text = product_model(csr).to_string()
    assert text == (GOLDEN / f"model_{name}.txt").read_text()
    back = ib.SpinModel.from_string(text)
    assert_same_csr(back.csr(), csr)
    assert back.layered == ((csr["layers"], csr["per_layer"]) if csr["layers"] else None)


@pytest.mark.parametrize("name", ["layered_12x5", "generic_mixed", "layered_8x4_zero_h"])
def test_reader_and_writer_agree_with_the_reference_library(lib, ref, name):
    csr = sample_csrs()[name]
    ref_model = ref.model(csr)
    text = ref_model.to_string()
    assert product_model(csr).to_string() == text
    # a shuffled document (edge lines reversed, CRLF, blank lines, decimal literal) loads to the same
    # canonical adjacency in both libraries
    lines = text.splitlines()
    head = [l for l in lines if not l.startswith("edge")]
    edges = [l for l in lines if l.startswith("edge")][::-1]
    shuffled = "\r\n".join(head + [""] + edges + ["  "]) + "\r\n"
    mine = ib.SpinModel.from_string(shuffled).csr()
    theirs = type(ref_model).from_string(ref, shuffled).csr()
    assert_same_csr(mine, theirs)
    assert_same_csr(mine, csr)


def test_file_round_trip_and_io_errors(lib, tmp_path):
    csr = sample_csrs()["layered_12x5"]
    model = product_model(csr)
    path = tmp_path / "m.ising"
    model.save(path)
    assert path.read_text() == model.to_string()
    assert_same_csr(ib.SpinModel.load(path).csr(), csr)
    with pytest.raises(ib.IsingError) as err:
        ib.SpinModel.load(tmp_path / "missing.ising")
    assert err.value.status == _lib.ISING_ERR_IO and "cannot open" in str(err.value)
    with pytest.raises(ib.IsingError) as err:
        model.save(tmp_path / "no_such_dir" / "m.ising")
    assert err.value.status == _lib.ISING_ERR_IO
    bad = tmp_path / "bad.ising"
    bad.write_text("ising-model v1\nspins 2\nedge 0 1 zzz space\n")
    with pytest.raises(ib.IsingError) as err:
        ib.SpinModel.load(bad)
    assert err.value.status == _lib.ISING_ERR_PARSE and f"{bad}: line 3: malformed edge line" in str(err.value)


HEADER = "ising-model v1\nspins 4\n"


@pytest.mark.parametrize("doc,message", [
    ("", "line 1: empty document, expected 'ising-model v1'"),
    ("ising-model v2\n", "line 1: expected header 'ising-model v1'"),
    ("ising-model v1\n", "line 1: missing spins line"),
    ("ising-model v1\nh 0 0x1p+0\n", "line 2: spins line must precede 'h'"),
    ("ising-model v1\nspins 0\n", "line 2: malformed spins line"),
    (HEADER + "spins 4\n", "line 3: duplicate spins line"),
    (HEADER + "layers 2 2\n", "line 3: layers * per_layer must equal spins with layers >= 4"),
    (HEADER + "layers 4\n", "line 3: malformed layers line"),
    (HEADER + "h 4 0x1p+0\n", "line 3: h index out of range"),
    (HEADER + "h 1 0x1p+0\n\nh 1 0x1p+1\n", "line 5: duplicate h line for spin 1"),
    (HEADER + "h 1 1.0x\n", "line 3: malformed h line"),
    (HEADER + "edge 1 0 0x1p+0 space\n", "line 3: edge endpoints must satisfy i < j"),
    (HEADER + "edge 0 9 0x1p+0 space\n", "line 3: edge endpoint out of range"),
    (HEADER + "edge 0 1 0x1p+0 space\nedge 0 1 0x1p+1 space\n", "line 4: duplicate edge 0-1"),
    (HEADER + "edge 0 1 0x1p+0 tau\n", "line 3: tau edge in a model without layers"),
    (HEADER + "edge 0 1 0x1p+0 diagonal\n", "line 3: malformed edge line"),
    (HEADER + "field 0 1\n", "line 3: unknown line 'field'"),
])
def test_parse_errors_name_the_line(lib, ref, doc, message):
    with pytest.raises(ib.IsingError) as err:
        ib.SpinModel.from_string(doc)
    assert err.value.status == _lib.ISING_ERR_PARSE
    assert str(err.value).endswith(message)
    if ref is not None:  # the reference rejects the same document with the same words
        with pytest.raises(ValueError) as theirs:
            ref.model(sample_csrs()["generic_mixed"]).from_string(ref, doc)
        assert str(theirs.value) == message


def test_structural_errors_after_parsing(lib):
    # four layers of one position, but spin 0 has a single tau edge: ISING_ERR_ARGUMENT, not PARSE
    doc = "ising-model v1\nspins 4\nlayers 4 1\nedge 0 1 0x1p+0 tau\n"
    with pytest.raises(ib.IsingError) as err:
        ib.SpinModel.from_string(doc)
    assert err.value.status == _lib.ISING_ERR_ARGUMENT and "tau edges, expected 2" in str(err.value)
