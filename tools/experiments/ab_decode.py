#!/usr/bin/env python3
"""Timing-only variants of the decode kernel for locating its bound (NOT parity-correct; never the product).

Copies paper_2506_09991_b200/csrc to a scratch dir, applies one textual patch per variant, builds
tools/ab/<variant>/libmvb200.so; run the bench against it with MV_LIB=tools/ab/<variant>/libmvb200.so.
  nopv     : the P.V issuer commits without issuing MMAs
  noqk     : the Q.K^T issuer commits without issuing MMAs (softmax then reads stale S)
  nosoft   : the softmax warps hand every S buffer straight back (no exp / P store)
  narrowF2 / narrowF4: units of <= 64 / <= 32 query rows replicated over 2 / 4 lane-quadrant copies (parity-checked
             candidates, not timing-only)
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
F2 = ("        w.copies = (rows > 32 && rows <= 64) ? 2 : 1;", "        w.copies = rows <= 64 ? 2 : 1;")
F4 = ("        w.copies = (rows > 32 && rows <= 64) ? 2 : 1;", "        w.copies = rows <= 32 ? 4 : (rows <= 64 ? 2 : 1);")
F4D = ("      if (copies == 2)\n        softmax_unit<2>", "      if (copies == 4)\n        softmax_unit<4>(P, g, n_ent, n_mem, se, warp, lane, tmem, s_full, p_full, vempty, xmax, m_ref, l);\n      else if (copies == 2)\n        softmax_unit<2>")
# timeline of CTA 0 (clock64), copied out with mv_debug_trace (tools/experiments/decode_timeline.py)
TR = "if (blockIdx.x == 0 && TRG < 256) g_mvtrace[(TRK) * 256 + TRG] = clock64();"
def tr(k, g="g"):
    return TR.replace("TRK", str(k)).replace("TRG", g)
TRACE = [
    ("namespace mv {\n\nnamespace {\n", "namespace mv {\n__device__ unsigned long long g_mvtrace[24 * 256];\nnamespace {\n"),
    ("    mbar_wait(&s_full[sb], (g / kSBufs) & 1);\n    tc::fence_after();\n    if (warp_active) {",
     "    mbar_wait(&s_full[sb], (g / kSBufs) & 1);\n    if (warp == 4 && lane == 0) { " + tr(0) + " if (blk == 0 && blockIdx.x == 0 && g < 256) g_mvtrace[16 * 256 + g] = 1; }\n    tc::fence_after();\n    if (warp_active) {"),
    ("      tc::tmem_wait_st();\n    }\n    tc::fence_before();\n    __syncwarp();\n    if (lane == 0) mbar_arrive(&p_full[sb]);",
     "      tc::tmem_wait_st();\n    }\n    tc::fence_before();\n    __syncwarp();\n    if (warp == 4 && lane == 0) { " + tr(3) + " }\n    if (lane == 0) mbar_arrive(&p_full[sb]);"),
    ("          if (g >= kSBufs) mbar_wait(&pv_done[sb], ((g - kSBufs) / kSBufs) & 1);  // P(g - kSBufs) consumed\n          mbar_wait(&kfull[sl], (g / kKSlots) & 1);",
     "          " + tr(4) + "\n          if (g >= kSBufs) mbar_wait(&pv_done[sb], ((g - kSBufs) / kSBufs) & 1);\n          " + tr(5) + "\n          mbar_wait(&kfull[sl], (g / kKSlots) & 1);\n          " + tr(6)),
    ("          mbar_wait(&p_full[sb], (g / kSBufs) & 1);\n          if (blk == 0 && i >= 1) mbar_wait(o_empty, (i - 1) & 1);  // epilogue drained O\n          mbar_wait(&vfull[g % kVSlots], (g / kVSlots) & 1);",
     "          mbar_wait(&p_full[sb], (g / kSBufs) & 1);\n          " + tr(7) + "\n          if (blk == 0 && i >= 1) mbar_wait(o_empty, (i - 1) & 1);\n          " + tr(8) + "\n          mbar_wait(&vfull[g % kVSlots], (g / kVSlots) & 1);\n          " + tr(9)),
    ("          if (g >= nsl) mbar_wait(&eb[sl], ((g / nsl) - 1) & 1);\n",
     "          if (is_k && sub == 0) " + tr(10) + "\n          if (g >= nsl) mbar_wait(&eb[sl], ((g / nsl) - 1) & 1);\n          if (is_k && sub == 0) " + tr(11) + "\n"),
    ("      constexpr uint32_t kFull = W == 32 ? 0xFFFFFFFFu : ((1u << W) - 1u);\n      tc::tmem_wait_ld();\n",
     "      constexpr uint32_t kFull = W == 32 ? 0xFFFFFFFFu : ((1u << W) - 1u);\n      tc::tmem_wait_ld();\n      if (warp == 4 && lane == 0) " + tr(17) + "\n"),
    ("      // the barrier also orders every warp's S reads before any warp's P / zero stores\n      if (group_any(bar_id, bar_cnt, need)) {",
     "      if (warp == 4 && lane == 0) " + tr(18) + "\n      const bool slow_ = group_any(bar_id, bar_cnt, need);\n      if (warp == 4 && lane == 0) " + tr(19) + "\n      if (slow_) {"),
    ("      l += ls;\n      tc::tmem_stNu<WP>(scol + part * WP, pk);", "      l += ls;\n      if (warp == 4 && lane == 0) " + tr(20) + "\n      tc::tmem_stNu<WP>(scol + part * WP, pk);"),
    ("      mbar_wait(stat_full, i & 1);\n", "      mbar_wait(stat_full, i & 1);\n      if (warp == 12 && lane == 0) " + tr(12, "i") + "\n"),
    ("      mbar_wait(o_full, i & 1);\n", "      mbar_wait(o_full, i & 1);\n      if (warp == 12 && lane == 0) " + tr(13, "i") + "\n"),
    ("      if (lane == 0) mbar_arrive(o_empty);\n", "      if (warp == 12 && lane == 0) " + tr(14, "i") + "\n      if (lane == 0) mbar_arrive(o_empty);\n"),
    ("extern \"C\" mv_status mv_attn_decode_plan_info(", "extern \"C\" MV_API int mv_debug_trace(void* host) { return (int)cudaMemcpyFromSymbol(host, mv::g_mvtrace, sizeof(mv::g_mvtrace)); }\nextern \"C\" mv_status mv_attn_decode_plan_info("),
]
SB3 = ("constexpr int kSBufs = 5;", "constexpr int kSBufs = 3;")
SB4 = ("constexpr int kSBufs = 5;", "constexpr int kSBufs = 4;")
NOEXP = ("""          const float2 pp = (kDecPoly > 0 && k % kDecPoly == kDecPoly - 1)
                                ? poly_exp2x2(xy)
                                : make_float2(fast_exp2(xy.x), fast_exp2(xy.y));""", "          const float2 pp = xy;")
ALLPOLY = ("""          const float2 pp = (kDecPoly > 0 && k % kDecPoly == kDecPoly - 1)""", """          const float2 pp = (true)""")
NOSTORE = ("      tc::tmem_stNu<WP>(scol + part * WP, pk);", "      if (pk[0] == 0x7fffffffu) tc::tmem_stNu<WP>(scol + part * WP, pk);")
POLY0 = ("constexpr int kDecPoly = 4;", "constexpr int kDecPoly = 0;")
POLY8 = ("constexpr int kDecPoly = 4;", "constexpr int kDecPoly = 8;")
POLY2 = ("constexpr int kDecPoly = 4;", "constexpr int kDecPoly = 2;")
VARIANTS = {"poly0": [POLY0], "poly8": [POLY8], "poly2": [POLY2], "noexp": [NOEXP], "allpoly": [ALLPOLY], "nostore": [NOSTORE], "sb3": [SB3], "sb4": [SB4], "trace": TRACE, "nopv": [PV], "noqk": [QK], "nosoft": [SOFT], "streamonly": [PV, QK, SOFT], "narrowF2": [F2],
            "narrowF4": [F4, F4D]}


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
