#!/usr/bin/env python3
"""Timing-only variants of the decode kernel for locating its bound (NOT parity-correct; never the product).

Copies paper_2506_09991_b200/csrc to a scratch dir, applies one textual patch per variant, builds
tools/ab/<variant>/libmvb200.so; run the bench against it with MV_LIB=tools/ab/<variant>/libmvb200.so.
  nopv     : the P.V issuer commits without issuing MMAs
  noqk     : the Q.K^T issuer commits without issuing MMAs (softmax then reads stale S)
  nosoft   : the softmax warps hand every S buffer straight back (no exp / P store)
  streamonly: noqk + nopv + nosoft: the K / V rings drain as fast as the TMA fills them
"""
import os
import pathlib
import shutil
import subprocess
import sys
import tempfile

REPO = pathlib.Path(__file__).resolve().parents[2]
CSRC = REPO / "paper_2506_09991_b200" / "csrc"

PV = ("          switch (sb) {\n            case 0: issue_pv_mmas<0>", "          if (false) switch (sb) {\n            case 0: issue_pv_mmas<0>")
QK = ("          switch (sb) {\n            case 0: issue_qk_mmas<0>", "          if (false) switch (sb) {\n            case 0: issue_qk_mmas<0>")
SOFT = ("    tc::fence_after();\n    if (warp_active) {\n      float v[W];", "    tc::fence_after();\n    if (false) {\n      float v[W];")
VARIANTS = {"nopv": [PV], "noqk": [QK], "nosoft": [SOFT], "streamonly": [PV, QK, SOFT]}


def build(name):
    out = REPO / "tools" / "ab" / name
    out.mkdir(parents=True, exist_ok=True)
    tmp = pathlib.Path(tempfile.mkdtemp())
    src = tmp / "csrc"
    shutil.copytree(CSRC, src)
    dec = src / "decode.cu"
    s = dec.read_text()
    for a, b in VARIANTS[name]:
        assert s.count(a) == 1, (name, a[:60])
        s = s.replace(a, b)
    dec.write_text(s)
    env = dict(os.environ, MV_BUILD_OUT=str(out / "libmvb200.so"), MV_BUILD_OBJ=str(out / "obj"))
    # build.py compiles CSRC: point it at the patched copy through a shim module
    code = (f"import importlib.util,pathlib,sys; spec=importlib.util.spec_from_file_location('b', '{REPO}/paper_2506_09991_b200/build.py');"
            f"m=importlib.util.module_from_spec(spec); spec.loader.exec_module(m); m.CSRC=pathlib.Path('{src}');"
            f"m.FLAGS=[f if not f.startswith('-I') or 'include' in f else '-I{src}' for f in m.FLAGS]; print(m.build())")
    subprocess.run([sys.executable, "-c", code], check=True, env=env)
    shutil.rmtree(tmp)


if __name__ == "__main__":
    for v in sys.argv[1:] or VARIANTS:
        build(v)
