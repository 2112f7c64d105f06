"""CPU-side checks of the drop-in boundary: the C-ABI library loads and exports every symbol
include/multiverse_b200.h declares (no compute calls: there is no GPU here)."""
import ctypes
import pathlib
import re
import subprocess

REPO = pathlib.Path(__file__).resolve().parent.parent
HEADER = REPO / "include" / "multiverse_b200.h"


def declared():
    return sorted(set(re.findall(r"^MV_API [^;(]*?\b(mv_\w+)\(", HEADER.read_text(), flags=re.M)))


def test_header_declares_the_path():
    names = declared()
    for must in ("mv_visibility", "mv_kv_fork", "mv_kv_merge", "mv_attn_decode", "mv_attn_prefill"):
        assert must in names


def test_library_exports_every_declared_symbol():
    import paper_2506_09991_b200 as m
    out = subprocess.run(["nm", "-D", "--defined-only", str(m.LIB_PATH)], capture_output=True, text=True).stdout
    exported = {line.split()[-1] for line in out.splitlines() if " T " in line}
    missing = [n for n in declared() if n not in exported]
    assert not missing, missing
    assert set(m.EXPORTED) == set(declared())
    assert {n for n in exported if n.startswith("mv_")} == set(declared())


def test_library_is_sm100a_and_version():
    import paper_2506_09991_b200 as m
    assert b"sm_100a" in m.lib.mv_version()
    sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", str(m.LIB_PATH)], capture_output=True,
                          text=True).stdout
    assert "sm_100a" in sass


def test_status_codes_mirror_reference_kinds():
    import paper_2506_09991_b200 as m
    assert m.CacheError.KINDS == {1: "UnknownHandle", 2: "DoubleRelease", 3: "CapacityExceeded",
                                  4: "BranchNotDescendant"}
    assert m.ParseError.KINDS == {5: "MalformedStructure", 6: "CountMismatch"}


def test_oracle_is_not_imported_by_the_product():
    for f in (REPO / "paper_2506_09991_b200").rglob("*"):
        if f.suffix in (".py", ".cu", ".cuh", ".hpp", ".cpp", ".h"):
            txt = f.read_text()
            assert "import oracle" not in txt and "from oracle" not in txt and "mv_oracle" not in txt, f
