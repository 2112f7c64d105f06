#!/usr/bin/env python3
"""Builds tools/ab/<name>/libmvb200.so with csrc/decode.cu (or csrc/<target>) replaced by <file> (A/B of whole
kernel versions; load one with MV_LIB=tools/ab/<name>/libmvb200.so).  usage: ab_files.py name=path.cu[@target.cu] ..."""
import os
import pathlib
import shutil
import subprocess
import sys
import tempfile

REPO = pathlib.Path(__file__).resolve().parents[2]
CSRC = REPO / "paper_2506_09991_b200" / "csrc"

for arg in sys.argv[1:]:
    name, path = arg.split("=", 1)
    path, target = (path.split("@", 1) + ["decode.cu"])[:2]
    out = REPO / "tools" / "ab" / name
    out.mkdir(parents=True, exist_ok=True)
    tmp = pathlib.Path(tempfile.mkdtemp())
    src = tmp / "csrc"
    shutil.copytree(CSRC, src)
    shutil.copy(path, src / target)
    env = dict(os.environ, MV_BUILD_OUT=str(out / "libmvb200.so"), MV_BUILD_OBJ=str(out / "obj"))
    code = (f"import importlib.util,pathlib; spec=importlib.util.spec_from_file_location('b', '{REPO}/paper_2506_09991_b200/build.py');"
            f"m=importlib.util.module_from_spec(spec); spec.loader.exec_module(m); m.CSRC=pathlib.Path('{src}');"
            f"m.FLAGS=[f if not f.startswith('-I') or 'include' in f else '-I{src}' for f in m.FLAGS]; print(m.build())")
    subprocess.run([sys.executable, "-c", code], check=True, env=env)
    shutil.rmtree(tmp)
