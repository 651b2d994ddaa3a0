"""CPU-side checks of the C-ABI boundary: the library loads without a GPU, exports every symbol
include/d360.h declares, the ctypes table matches the header, and the product never falls back
to (or imports) the oracle."""
import ctypes
import re
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

HEADER = ROOT / "include" / "d360.h"


def declared_symbols():
    text = re.sub(r"/\*.*?\*/", "", HEADER.read_text(), flags=re.S)
    return sorted(set(re.findall(r"\b(d360_[a-z0-9_]+)\s*\(", text)))


@pytest.fixture(scope="module")
def built():
    from paper_2211_16266_b200 import _build

    return _build.build()


def test_library_exports_every_declared_symbol(built):
    lib = ctypes.CDLL(str(built))
    syms = declared_symbols()
    assert len(syms) >= 20
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing


def test_ctypes_table_matches_header(built):
    from paper_2211_16266_b200 import _lib

    assert sorted(_lib.EXPORTED_SYMBOLS) == declared_symbols()
    handle = _lib.load()  # sets restype / argtypes for every entry; raises BackendError if one is absent
    assert handle.d360_version() >= 100
    assert _lib.launch_count() == 0  # nothing launched by loading


def test_header_cites_the_reference_interface():
    text = HEADER.read_text()
    for fn, cite in [("d360_eval_costs", "K:300-349"), ("d360_red_black_pass", "K:352-473"),
                     ("d360_refine_pass", "K:476-610"), ("d360_median_support_mask", "K:613-647"),
                     ("d360_run_patchmatch", "E:563-631"), ("d360_warp_plane_map", "E:286-355"),
                     ("d360_random_init", "E:244-283"), ("d360_consistency_filter", "P:246-281"),
                     ("d360_fuse_oldest", "P:310-348")]:
        i = text.index(f"int {fn}(")
        assert cite in text[max(0, i - 1200):i], (fn, cite)


def test_group_struct_layout_matches_header(built):
    """sizeof / field order of d360_group as compiled by gcc == the ctypes Structure."""
    from paper_2211_16266_b200 import _lib

    src = '#include <stdio.h>\n#include <stddef.h>\n#include "d360.h"\nint main(void){printf("%zu %zu %zu %zu %zu\\n",' \
          'sizeof(d360_group), offsetof(d360_group, rays), offsetof(d360_group, nb_pad_x), ' \
          'offsetof(d360_group, rel_r), offsetof(d360_group, trunc));return 0;}'
    exe = Path("/tmp/d360_layout_check")
    subprocess.run(["gcc", "-x", "c", "-", f"-I{HEADER.parent}", "-o", str(exe)], input=src.encode(), check=True)
    got = [int(x) for x in subprocess.run([str(exe)], capture_output=True, check=True).stdout.split()]
    G = _lib.Group
    assert got == [ctypes.sizeof(G), G.rays.offset, G.nb_pad_x.offset, G.rel_r.offset, G.trunc.offset]


def test_no_cpu_fallback_and_no_oracle_import():
    from paper_2211_16266_b200 import engine
    from paper_2211_16266_b200.errors import BackendError

    import torch

    if not torch.cuda.is_available():
        with pytest.raises(BackendError):
            engine.to_gray(__import__("numpy").zeros((4, 8, 3), "uint8"))
    pkg = ROOT / "paper_2211_16266_b200"
    for path in pkg.rglob("*.py"):
        assert "oracle" not in path.read_text().replace("oracle/", ""), f"{path} mentions the oracle"


@pytest.mark.parametrize("name", ["hot_64x32_ident", "hot_64x32_rot", "hot_256x128_c1"])
def test_refinement_draw_tables_equal_the_reference(name):
    """engine.refinement_draw_tables (host logic, E:495-526) reproduces the tables the reference drew
    for the golden runs, bit for bit (same PCG64 stream, same draw order, same f32 rounding)."""
    import numpy as np

    from paper_2211_16266_b200 import engine

    z = np.load(ROOT / "tests" / "golden" / f"{name}.npz")
    dr = z["depth_range"]
    got = engine.refinement_draw_tables(int(z["seed"]), int(z["iterations"]), 0.25 * (dr[1] - dr[0]), np.deg2rad(60.0))
    assert got.dtype == np.float32 and np.array_equal(got, z["tables"])


def test_integration_md_group_struct_matches_ctypes_table():
    """The Group structure printed in INTEGRATION.md (what a maintainer would paste) has the fields of
    the library's own ctypes table, in order."""
    from paper_2211_16266_b200 import _lib

    text = (ROOT / "INTEGRATION.md").read_text()
    block = re.search(r"class Group\(C\.Structure\):.*?_fields_ = \[(.*?)\]\n", text, re.S).group(1)
    names = re.findall(r'\("(\w+)"', block)
    assert names == [f[0] for f in _lib.Group._fields_]
