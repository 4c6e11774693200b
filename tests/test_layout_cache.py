"""On-disk and in-process layout caches (sgx_layout_io.cpp, sgx_api.cpp
layoutcache), host only.  A layout read back from disk must equal the
compiled one in every persisted field (sgx_layout_digest); damaged or foreign
files are rejected and the layout recompiled; the key covers the layout's
environment knobs."""
import os

import pytest

from paper_2502_08673_b200 import layout_digest, load_instance, set_layout_cache_dir


@pytest.fixture
def cache_dir(tmp_path, monkeypatch):
    monkeypatch.setenv("SGX_NO_LAYOUT_CACHE", "1")  # disk only: every lookup reaches the file
    set_layout_cache_dir(str(tmp_path))
    yield tmp_path
    set_layout_cache_dir(None)


@pytest.mark.parametrize("name", ["c3a_or50", "c2_iscas", "c4_blasted"])
def test_disk_round_trip_equals_compiled(cache_dir, name):
    inst = load_instance(name)
    built, src = layout_digest(inst.cnf, inst.circuit, inst.paths)
    assert src == 0
    files = list(cache_dir.glob("*.sgxlayout"))
    assert len(files) == 1 and files[0].stat().st_size > 0
    loaded, src = layout_digest(inst.cnf, inst.circuit, inst.paths)
    assert src == 2 and loaded == built


def test_damaged_file_is_recompiled(cache_dir):
    inst = load_instance("c3a_or50")
    built, _ = layout_digest(inst.cnf, inst.circuit, inst.paths)
    (f,) = cache_dir.glob("*.sgxlayout")
    data = f.read_bytes()
    f.write_bytes(data[: len(data) // 2])  # truncated
    again, src = layout_digest(inst.cnf, inst.circuit, inst.paths)
    assert src == 0 and again == built
    f.write_bytes(b"XXXXXXXX" + data[8:])  # wrong magic
    again, src = layout_digest(inst.cnf, inst.circuit, inst.paths)
    assert src == 0 and again == built
    again, src = layout_digest(inst.cnf, inst.circuit, inst.paths)  # rewritten intact
    assert src == 2 and again == built


def test_key_covers_circuit_and_knobs(cache_dir, monkeypatch):
    a, b = load_instance("c3a_or50"), load_instance("c3b_or100")
    da, _ = layout_digest(a.cnf, a.circuit, a.paths)
    db, src = layout_digest(b.cnf, b.circuit, b.paths)
    assert src == 0 and db != da
    monkeypatch.setenv("SGX_ALL_CLAUSES", "1")  # a different harvest program: a different key
    dk, src = layout_digest(a.cnf, a.circuit, a.paths)
    assert src == 0 and dk != da
    assert len(list(cache_dir.glob("*.sgxlayout"))) == 3


def test_in_process_cache(monkeypatch):
    monkeypatch.delenv("SGX_NO_LAYOUT_CACHE", raising=False)
    set_layout_cache_dir(None)
    inst = load_instance("c1b_random")
    d0, _ = layout_digest(inst.cnf, inst.circuit, inst.paths)
    d1, src = layout_digest(inst.cnf, inst.circuit, inst.paths)
    assert src == 1 and d1 == d0
