"""C-ABI boundary checks that need no GPU: the library builds for sm_100a,
loads, exports every symbol include/atos.h declares, and the ctypes mirror
structs match the C layout."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "include", "atos.h")


@pytest.fixture(scope="module")
def lib():
    from paper_2112_00132_b200 import build
    build.build()
    import paper_2112_00132_b200 as atos
    return atos


def _declared():
    src = open(HDR).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(atos_[a-z_]+)\s*\(", src)))


def test_exports_every_declared_symbol(lib):
    L = lib.lib()
    names = _declared()
    assert "atos_bfs" in names and "atos_graph_create" in names
    for s in names:
        assert hasattr(L, s), s
    assert set(lib.EXPORTS) == set(names)


def test_sm100a_code_present(lib):
    out = subprocess.run(["cuobjdump", "--list-elf", lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_struct_layout_matches_c(lib, tmp_path):
    c = tmp_path / "sz.c"
    c.write_text('#include "atos.h"\n#include <stdio.h>\n#include <stddef.h>\n'
                 'int main(){printf("%zu %zu %zu %zu %zu\\n", sizeof(atos_config), sizeof(atos_stats),'
                 ' offsetof(atos_config, stream), offsetof(atos_stats, max_residue), offsetof(atos_config, timeout_s));}')
    exe = tmp_path / "sz"
    subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), "-o", str(exe), str(c)])
    got = list(map(int, subprocess.check_output([str(exe)]).split()))
    assert got == [ctypes.sizeof(lib.CConfig), ctypes.sizeof(lib.CStats), lib.CConfig.stream.offset,
                   lib.CStats.max_residue.offset, lib.CConfig.timeout_s.offset]


def test_host_only_entry_points(lib):
    L = lib.lib()
    cfg = lib.CConfig()
    L.atos_config_default(ctypes.byref(cfg))
    assert cfg.struct_size == ctypes.sizeof(lib.CConfig)
    assert cfg.worker == 2 and cfg.kernel == 0 and cfg.fetch_size == 256
    assert L.atos_status_string(6) == b"ATOS_ERR_QUEUE_OVERFLOW"
    assert lib.version().startswith("atos-b200")
    # argument validation happens before any device work
    h = ctypes.c_void_p()
    assert L.atos_graph_create(None, None, -1, 0, 0, ctypes.byref(h)) == 1
    assert L.atos_graph_create(None, None, 0, 0, 0, None) == 1
    assert L.atos_bfs(None, 0, None, None, None) == 1
    # bits 30-31 of a column entry are tags (R37): n >= 2^30 - 1 is UNSUPPORTED, refused before any read
    one = (ctypes.c_int64 * 1)(0)
    assert L.atos_graph_create(one, None, 2 ** 30 - 1, 0, 0, ctypes.byref(h)) == 8
    assert L.atos_graph_create_peer(2, None, one, None, 2 ** 30 - 1, 0, 0, ctypes.byref(h)) == 8
    assert L.atos_graph_create_peer(0, None, one, None, 4, 0, 0, ctypes.byref(h)) == 1


def test_product_has_no_oracle_dependency():
    """The CUDA path shares no code with oracle/ and never imports it."""
    pkg = os.path.join(ROOT, "paper_2112_00132_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dp, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt and "oracle.c" not in txt, f
    for f in os.listdir(os.path.join(ROOT, "oracle")):
        if f.endswith((".py", ".c")):
            txt = open(os.path.join(ROOT, "oracle", f)).read()
            assert "import paper_2112_00132_b200" not in txt and "from paper_2112_00132_b200" not in txt, f
