"""Grid I/O of the drop-in, CPU only.

Re-expresses the reference's I/O tests (proj/tests/test_io_cli.cpp:62-115)
against fsx_write_grid / fsx_read_grid (csrc/fsx_io.cpp), plus the sidecar
validation of proj/src/grid_io.cpp:133-180 and run_bench's table layout
(proj/src/runner.cpp:46-62)."""
import os

import numpy as np
import pytest

import paper_2105_06676_b200 as fs
import refutil as R


def test_raw_round_trip_is_bit_exact(tmp_path):
    """test_io_cli.cpp:62-70"""
    rng = R.Rng(167)
    g = fs.FieldGrid(fs.GridShape([4, 4], 2), R.random_grid(rng, 32))
    p = str(tmp_path / "fftstencil_test_grid.raw")
    fs.write_grid(g, p, "raw")
    back = fs.read_grid(p)
    assert back.shape.dims() == [4, 4] and back.shape.fields() == 2
    assert np.array_equal(back.data, g.data)
    assert open(p + ".meta").read() == "dims = 4 4\nfields = 2\ndtype = float64\norder = row-major\n"
    assert os.path.getsize(p) == 32 * 8
    assert np.array_equal(np.fromfile(p, dtype="<f8"), g.data)  # little-endian, row-major then field


def test_csv_matches_the_documented_two_cell_example(tmp_path):
    """test_io_cli.cpp:72-88"""
    g = fs.FieldGrid(fs.GridShape([2]), np.array([1.5, -2.0]))
    p = str(tmp_path / "fftstencil_test_grid.csv")
    fs.write_grid(g, p, "csv")
    assert open(p).read().splitlines()[:2] == ["0,0,1.5", "1,0,-2"]
    back = fs.read_grid(p)
    assert back.shape.dims() == [2] and np.array_equal(back.data, g.data)


def test_csv_round_trip_on_awkward_values(tmp_path):
    """test_io_cli.cpp:90-97: shortest round-trip decimals"""
    vals = np.array([1.0 / 3.0, -0.1, 1e-300, 7.000000000000001, 0.0, -12345.6789])
    g = fs.FieldGrid(fs.GridShape([3], 2), vals)
    p = str(tmp_path / "fftstencil_test_grid2.csv")
    fs.write_grid(g, p, "csv")
    assert np.array_equal(fs.read_grid(p).data, vals)


def test_truncated_raw_file_reports_the_byte_counts(tmp_path):
    """test_io_cli.cpp:99-106"""
    g = fs.FieldGrid(fs.GridShape([8]), R.random_grid(R.Rng(173), 8))
    p = str(tmp_path / "fftstencil_test_trunc.raw")
    fs.write_grid(g, p, "raw")
    os.truncate(p, 8 * 8 - 3)
    with pytest.raises(fs.IoError, match="expected 64 bytes"):
        fs.read_grid(p)


def test_malformed_csv_names_the_line(tmp_path):
    """test_io_cli.cpp:108-115"""
    p = str(tmp_path / "fftstencil_test_bad.csv")
    with open(p, "w") as f:
        f.write("0,0,1.5\nnot,a,number\n")
    with pytest.raises(fs.IoError, match=":2"):
        fs.read_grid(p)


@pytest.mark.parametrize("meta,msg", [
    ("dims = 4\nfields = 1\ndtype = float32\norder = row-major\n", "unsupported dtype 'float32'"),
    ("dims = 4\nfields = 1\ndtype = float64\norder = col-major\n", "unsupported order 'col-major'"),
    ("dims = 4\nfields = 1\nzzz = 1\n", "unknown key 'zzz'"),
    ("fields = 1\ndtype = float64\n", "missing dims or fields"),
    ("dims 4\n", "expected 'key = value'"),
])
def test_raw_sidecar_validation(tmp_path, meta, msg):
    """proj/src/grid_io.cpp:133-170"""
    p = str(tmp_path / "g.raw")
    np.zeros(4).tofile(p)
    with open(p + ".meta", "w") as f:
        f.write(meta)
    with pytest.raises(fs.IoError, match=msg):
        fs.read_grid(p)


def test_csv_errors(tmp_path):
    """proj/src/grid_io.cpp:52-110: column count, duplicates, missing values, non-finite"""
    cases = {"cols.csv": ("0,0,1\n1,0,0,2\n", "inconsistent column count"),
             "dup.csv": ("0,0,1\n0,0,2\n2,0,3\n", "duplicate cell"),
             "count.csv": ("0,0,1\n2,0,2\n", "got 2 lines for a grid of 3 values"),
             "nan.csv": ("0,0,nan\n", "non-finite value"),
             "empty.csv": ("\n", "empty grid file")}
    for name, (text, msg) in cases.items():
        p = str(tmp_path / name)
        with open(p, "w") as f:
            f.write(text)
        with pytest.raises(fs.IoError, match=msg):
            fs.read_grid(p)
    with pytest.raises(fs.IoError, match="cannot open"):
        fs.read_grid(str(tmp_path / "missing.csv"))


def test_multidim_csv_order(tmp_path):
    """row-major cells, field innermost; read back any line order"""
    g = fs.FieldGrid(fs.GridShape([2, 3], 2), np.arange(12.0) - 5.5)
    p = str(tmp_path / "m.csv")
    fs.write_grid(g, p, "csv")
    lines = open(p).read().splitlines()
    assert lines[0] == "0,0,0,-5.5" and lines[1] == "0,0,1,-4.5" and lines[2] == "0,1,0,-3.5"
    with open(p, "w") as f:
        f.write("\n".join(reversed(lines)) + "\n")
    back = fs.read_grid(p)
    assert back.shape.dims() == [2, 3] and back.shape.fields() == 2 and np.array_equal(back.data, g.data)


def test_stage_table_layout():
    """runner.cpp:46-62: every stage, total, optional naive_total, fixed 6 decimals"""
    st = fs.StageTimings()
    st.forward_fft, st.squaring, st.inverse_fft = 0.25, 0.125, 0.5
    text = fs.format_stage_table(st, 1.0)
    lines = text.splitlines()
    assert lines[0] == "stage timings (seconds):"
    assert lines[1] == "  forward_fft         0.250000"
    assert [ln.split()[0] for ln in lines[1:]] == ["forward_fft", "squaring", "hadamard", "inverse_fft",
                                                   "boundary_recursion", "total"]
    assert "naive_total" in fs.format_stage_table(st, 1.0, 2.5)
