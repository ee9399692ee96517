"""SFSV container format (CPU): the fixture writer against the reference's own
save_volume, and load_volume's error codes for the malformed variants that
sfseg_load_files must reproduce (tests/test_gpu_files.py)."""
import numpy as np
import pytest

from paper_1907_02731_b200 import engine as E
from tests import sfsv_util as U
from tests.oracle_lib import Reference, random_volume, reference_available

pytestmark = pytest.mark.skipif(not reference_available(), reason="oracle/_ref not built")


def test_writer_matches_reference_save_volume(tmp_path):
    v = random_volume((3, 7, 11), 5)
    Reference().save_volume(tmp_path / "ref.sfsv", v)
    U.write(tmp_path / "ours.sfsv", v)
    assert (tmp_path / "ref.sfsv").read_bytes() == (tmp_path / "ours.sfsv").read_bytes()
    assert E.volume_shape(tmp_path / "ref.sfsv") == (3, 7, 11)


def test_reference_load_volume_error_codes(tmp_path):
    v = random_volume((2, 5, 9), 6)
    for name, path, code in U.malformed_cases(tmp_path, v):
        rc, _ = Reference().load_volume_rc(path)
        assert rc == code, f"{name}: reference load_volume status {rc}, fixture expects {code}"
    U.write(tmp_path / "ok.sfsv", v)
    assert Reference().load_volume_rc(tmp_path / "ok.sfsv") == (0, (2, 5, 9))
