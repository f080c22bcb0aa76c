"""CPU-side checks of the drop-in boundary: the C-ABI library loads, exports
every entry point include/catgnn.h declares, and its host-only parts (artifact
reader, replica map, replication factor, error codes) match the reference.
No kernel is launched here."""
import ctypes as C
import os
import re

import numpy as np
import pytest

from oracle import ref

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    src = open(os.path.join(ROOT, "include", "catgnn.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(catgnn_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_header_symbol():
    from paper_2404_02300_b200 import _lib
    lib = C.CDLL(_lib.LIB_PATH)
    names = header_functions()
    assert len(names) > 40
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_library_is_sm100a():
    so = os.path.join(ROOT, "paper_2404_02300_b200", "libcatgnn.so")
    data = open(so, "rb").read()
    assert b"sm_100a" in data


def test_artifact_reader_matches_reference(small_ds, small_artifact):
    from paper_2404_02300_b200 import gnnpart as gp
    art = gp.Artifact(small_artifact)
    rf, mrf = ref.artifact_replication_factor(small_artifact)
    # RF bit-exact: the same f64 division over the same record counts
    assert gp.replication_factor(art) == rf
    assert art.info.manifest_replication_factor == mrf
    assert art.info.num_nodes == small_ds["n"]
    assert art.info.num_edges == small_ds["edges"].shape[0]
    total = 0
    owners = {}
    for s in range(art.num_partitions):
        ext, own, role, home = art.replica_map(s)
        total += ext.size
        assert np.all(np.diff(ext.astype(np.int64)) > 0)          # ascending ext id
        assert np.all(home[own == 1] == s)                       # owners are home
        assert np.all(home[own == 0] != s)                       # halo rows live elsewhere
        assert np.all(role[own == 0] == 0)                       # roles on owners only
        np.testing.assert_array_equal(role[own == 1], small_ds["roles"][ext[own == 1].astype(np.int64)])
        for x in ext[own == 1]:
            owners[int(x)] = s
    assert len(owners) == small_ds["n"]
    for s in range(art.num_partitions):
        ext, own, _, home = art.replica_map(s)
        assert all(owners[int(x)] == h for x, h in zip(ext, home))


def test_artifact_errors_mirror_reference(tmp_path, small_artifact):
    from paper_2404_02300_b200 import gnnpart as gp
    with pytest.raises(gp.DataError, match="missing manifest"):
        gp.Artifact(str(tmp_path / "nope"))
    # corrupt an edge file: truncated record -> DataError (edge_stream.cpp:47-48)
    import shutil
    bad = tmp_path / "bad"
    shutil.copytree(small_artifact, bad)
    with open(bad / "part-0" / "edges.bin", "ab") as f:
        f.write(b"\x01\x02\x03")
    with pytest.raises(gp.DataError, match="truncated record"):
        gp.Artifact(str(bad))
    with pytest.raises(ref.RefError) as e:
        ref.artifact_replication_factor(str(bad))
    assert e.value.code == 3
    # count mismatch -> "corrupt artifact"
    bad2 = tmp_path / "bad2"
    shutil.copytree(small_artifact, bad2)
    lines = open(bad2 / "part-1" / "nodes.tsv").read().splitlines()
    open(bad2 / "part-1" / "nodes.tsv", "w").write("\n".join(lines[:-1]) + "\n")
    with pytest.raises(gp.DataError, match="corrupt artifact"):
        gp.Artifact(str(bad2))


def test_sync_weights_matches_reference():
    from paper_2404_02300_b200 import gnnpart as gp
    for counts in ([1, 3], [5, 0], [7, 11, 13], [1, 1, 1]):
        assert np.array_equal(gp.sync_weights(counts), ref.sync_weights(counts))
    with pytest.raises(gp.DataError):
        gp.sync_weights([0, 0])


def test_context_fails_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2404_02300_b200 import gnnpart as gp
    with pytest.raises(gp.InternalError):
        gp.Context(0)
