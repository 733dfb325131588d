"""Host-side MatrixMarket header parsing of the ingest path (no GPU)."""
import io

import numpy as np
import pytest
import scipy.io as sio
import scipy.sparse as sp

from paper_2605_13928_b200.ingest import mtx_header


def _raw(text: str) -> np.ndarray:
    return np.frombuffer(text.encode(), dtype=np.uint8)


def test_header_from_scipy_writer():
    M = sp.random(50, 30, density=0.1, format="coo", random_state=1)
    for field, code in (("integer", 0), ("real", 1), ("pattern", 2)):
        b = io.BytesIO()
        sio.mmwrite(b, M, field=field)
        raw = np.frombuffer(b.getvalue(), np.uint8)
        h = mtx_header(raw)
        assert (h.field, h.n_rows, h.n_cols, h.nnz) == (code, 50, 30, M.nnz)
        first = bytes(raw[h.data_offset:h.data_offset + 40]).decode().split("\n")[0].split()
        assert len(first) == (2 if field == "pattern" else 3)


def test_header_comments_and_blank_lines():
    h = mtx_header(_raw("%%MatrixMarket matrix coordinate real general\n% c1\n%\n\n 3 4 2\n1 1 1.5\n2 3 -2e3\n"))
    assert (h.field, h.n_rows, h.n_cols, h.nnz) == (1, 3, 4, 2)
    assert bytes(_raw("x")).decode() == "x"


@pytest.mark.parametrize("text", [
    "%%MatrixMarket matrix array real general\n2 2\n1\n2\n3\n4\n",
    "%%MatrixMarket matrix coordinate complex general\n1 1 1\n1 1 1 0\n",
    "%%MatrixMarket matrix coordinate real symmetric\n2 2 1\n1 1 1\n",
    "%%NotMatrixMarket\n",
    "%%MatrixMarket matrix coordinate real general\n% only comments\n",
])
def test_header_rejects(text):
    with pytest.raises(ValueError):
        mtx_header(_raw(text))
