"""Generate the kernel-instantiation translation units and the registry.

Run by the build (``make -C paper_2305_07390_b200/csrc``); outputs are
committed so the tree builds without Python too.  One translation unit per
(shape, exactness) keeps nvcc parallel (``make -j``).
"""

from __future__ import annotations

import os

HERE = os.path.dirname(os.path.abspath(__file__))

# shape id, C++ type, tag, list of (T, C)
S2D = [
    ("SHAPE_J2D5PT", "StarShape<2, 1>", "j2d5pt",
     [(t, 4 if t <= 10 else 2) for t in range(1, 17)]),
    ("SHAPE_J2D9PT_GOL", "BoxShape<2, 1>", "j2d9pt_gol", [(t, 4) for t in (1, 2, 3, 4, 6, 8)]),
    ("SHAPE_J2D9PT", "StarShape<2, 2>", "j2d9pt", [(t, 4) for t in (1, 2, 3, 4, 5)]),
    ("SHAPE_J2D25PT", "BoxShape<2, 2>", "j2d25pt", [(t, 4) for t in (1, 2, 3, 4)]),
    ("SHAPE_J2D13PT", "StarShape<2, 3>", "j2d13pt", [(t, 4) for t in (1, 2, 3)]),
    ("SHAPE_J2DS25PT", "StarShape<2, 6>", "j2ds25pt", [(t, 4) for t in (1, 2)]),
]
NW, S = 4, 8
# shifted-window 2-D kernels for large radii (see stream2d_unit), registered
# FIRST so they are the planner default: j2ds25pt 196 -> 240 GCells/s at t=1
# (R = 3 measured slower shifted, 527 vs 487, and keeps rotating windows)
SHIFT_2D = {"j2ds25pt": [(1, 4, 4), (2, 4, 4)]}  # (t, C, U): U=4 251, U=1 240, U=2 226 GCells/s
# (R = 3 with U = 4 shifted windows measured 480 / 531 vs rotating 530 / 552: rotating)
SHIFT_2D_AFTER = {}  # shifted variants registered after the rotating kernels

# tolerance-mode (exact = 0) kernels for uniform coefficients: reassociated
# tap sums (stream2d_unit's block_ra, shifted windows of 4 rows, 4 cells per
# lane): (T, MINB, SHIFT, S) -- SHIFT 4: level-major shifted windows (shared
# column sums of 4 targets, large radii), 0: rotating windows
RA_2D = {"j2ds25pt": [(1, 2, 4, 16)],
         "j2d13pt": [(2, 2, 0, 8), (1, 2, 4, 16), (3, 2, 0, 8)],
         "j2d25pt": [(3, 2, 0, 8), (1, 2, 0, 16), (2, 2, 0, 8)],
         "j2d9pt_gol": [(6, 2, 0, 8), (1, 2, 0, 16), (2, 2, 0, 8), (3, 2, 0, 8), (4, 2, 0, 8)],
         "j2d9pt": [(3, 2, 0, 8), (1, 2, 0, 16), (2, 2, 0, 8)]}

# tolerance-mode halo-exchange kernels (halo2d_unit's block_ra, stars with
# R >= 4): (T, C, MINB, S)
RA_H2D = {"j2ds25pt": [(1, 4, 1, 16), (2, 2, 1, 16)]}

# 3-D: shape id, C++ type, tag, list of (T, CY, CX, NWY, S, DEC, MINB); the first
# entry per depth is the planner default.
S3D = [
    ("SHAPE_J3D7PT", "StarShape<3, 1>", "j3d7pt",
     [(1, 4, 2, 8, 4, 0, 1), (2, 4, 2, 8, 4, 0, 1), (3, 4, 2, 8, 4, 0, 1), (4, 4, 2, 8, 4, 0, 1),
      (2, 2, 2, 16, 4, 0, 1), (3, 2, 2, 16, 4, 0, 1)]),
# (taller one-CTA tiles measured and dropped: 9-13 warps get <= 168 registers
# per thread (3 warps per SMSP) and spill -- t=4 x 10 warps 269, x 9 warps 321,
# t=3 x 12 warps 482, x 13 warps 295 vs 681 / 701 for 8 warps; a taller tile
# needs a second SM's registers: the 2-CTA cluster kernel)
    ("SHAPE_J3D13PT", "StarShape<3, 2>", "j3d13pt", [(1, 4, 2, 8, 4, 0, 1), (2, 4, 2, 8, 4, 0, 1)]),
    ("SHAPE_J3D27PT", "BoxShape<3, 1>", "j3d27pt",
     [(1, 4, 2, 8, 4, 0, 1), (2, 4, 2, 8, 4, 0, 1), (1, 2, 2, 16, 4, 0, 1), (2, 2, 2, 16, 4, 0, 1)]),
    # plane-major partial sums (stream3d_unit_pm): 4x2 cells fit without spills
    ("SHAPE_J3D17PT", "NoCornerShape3<true>", "j3d17pt", [(1, 4, 2, 8, 4, 0, 1), (2, 4, 2, 8, 4, 0, 1)]),
    ("SHAPE_POISSON", "NoCornerShape3<false>", "poisson", [(1, 4, 2, 8, 4, 0, 1), (2, 4, 2, 8, 4, 0, 1)]),
]

# tolerance-mode (exact = 0) kernels for uniform coefficients: reassociated
# tap sums (stream3d_unit_pm's pattern sums), same tile configs as "u"
RA_3D = {"j3d27pt": [(2, 4, 2, 8, 4, 0, 1), (1, 4, 2, 8, 4, 0, 1)],
         "poisson": [(2, 4, 2, 8, 4, 0, 1), (1, 4, 2, 8, 4, 0, 1)],
         "j3d17pt": [(2, 4, 2, 8, 4, 0, 1), (1, 4, 2, 8, 4, 0, 1)]}

# 2-CTA cluster kernels (ebisu_stream3d_cl.cuh: one 64x64 tile over two SMs,
# DSMEM seam exchange), shared-product fp64: (T, CY, CX, NWY, S); registered
# after the one-CTA kernels of the same depth (opt-in variants).  Measured
# (512^3 x 500): t=3 601 / t=2 497 GCells/s vs 701 / 585 for one CTA despite
# V 0.72 vs 0.65 -- the pair runs at the pace of its slower SM every advance;
# t=4 does not fit the register file with the seam state (424 B spills, 372)
CL3D = {"j3d7pt": [(3, 4, 2, 8, 4), (2, 4, 2, 8, 4)]}

# fp32 (north-star 1e-5 mode), shared-product kernels only (uniform
# coefficients; other stencils run the fp32 naive kernel).  Floats halve the
# window registers, so 2-D strips are 32*8 = 256 columns wide (the TMA box
# limit) at the same register cost as fp64 with 4 cells per lane.
# (depths 1 and 2 of every shape keep sweep remainders on the TB kernels)
F32_2D = {"j2d5pt": [(4, 8), (8, 8), (12, 4), (16, 4), (1, 8), (2, 8)],
          "j2d9pt_gol": [(2, 8), (1, 8)], "j2d9pt": [(2, 8), (1, 8)], "j2d25pt": [(2, 4), (1, 4)],
          "j2d13pt": [(2, 4), (1, 4)], "j2ds25pt": [(1, 4)]}
# fp32 3-D: half the registers -> 12-warp 48x64 tiles (t=4: 1284 vs 1151
# GCells/s with 8 warps; t=5/6 and 4x4-cell tiles measured slower)
F32_3D = {"j3d7pt": [(4, 4, 2, 12, 4, 0, 1), (3, 4, 2, 12, 4, 0, 1), (2, 4, 2, 8, 4, 0, 1),
                     (4, 4, 2, 8, 4, 0, 1), (1, 4, 2, 8, 4, 0, 1)],
          "j3d27pt": [(1, 4, 2, 8, 4, 0, 1), (2, 4, 2, 8, 4, 0, 1)],
          "j3d13pt": [(1, 4, 2, 8, 4, 0, 1)], "j3d17pt": [(1, 4, 2, 8, 4, 0, 1)],
          "poisson": [(1, 4, 2, 8, 4, 0, 1)]}

# 2-D halo exchange (device tiling): shape id, C++ type, tag, list of (T, C);
# 8 warps per CTA strip
H2D = [
    ("SHAPE_J2D5PT", "StarShape<2, 1>", "j2d5pt", [(4, 4), (6, 2), (8, 2), (12, 2), (16, 2)]),
    ("SHAPE_J2D9PT_GOL", "BoxShape<2, 1>", "j2d9pt_gol", [(2, 4), (4, 4)]),
    ("SHAPE_J2D9PT", "StarShape<2, 2>", "j2d9pt", [(2, 4), (4, 4)]),
    ("SHAPE_J2D25PT", "BoxShape<2, 2>", "j2d25pt", [(2, 4), (3, 4)]),
    ("SHAPE_J2D13PT", "StarShape<2, 3>", "j2d13pt", [(1, 4), (2, 4), (3, 4), (4, 2)]),
    ("SHAPE_J2DS25PT", "StarShape<2, 6>", "j2ds25pt", [(1, 4), (2, 2), (3, 2), (4, 2)]),
]
H2D_NW, H2D_S = 8, 8
SHIFT_H2D = {"j2ds25pt": [(1, 4, 4), (2, 2, 4)]}  # (t, C, U): U=4 169 / 170, U=1 151 / 145
# (halo j2d13pt with U=4 shifted windows: 311 / 323 vs rotating 326 / 351: rotating)
SHIFT_H2D_AFTER = {}  # shifted variants registered after the rotating kernels
# cluster-tile twins (device tiles of several CTAs exchanging seams through
# DSMEM), bitwise shared-product kernels: (t, C, shift)
H2D_CLU = {"j2d5pt": [(4, 4, 0), (8, 2, 0)], "j2d9pt_gol": [(2, 4, 0)], "j2d9pt": [(2, 4, 0)],
           "j2d25pt": [(2, 4, 0)], "j2d13pt": [(2, 4, 0), (3, 4, 0)],
           "j2ds25pt": [(1, 4, 4), (2, 2, 4)]}


def h2d_minb(t, r, c, star):
    w = (max(r, 2) + r + 1) if star else (2 * r + 2)
    est = 2 * t * w * c + 72
    return max(1, min(4, 65536 // (H2D_NW * 32 * max(est, 64))))


HEADER = "// GENERATED by gen_instances.py -- do not edit.\n"


def _trim_fma(cfgs, dims):
    """FMA-mode per-tap kernels only serve non-uniform coefficients; keep a few depths."""
    if dims == 2:
        keep = [c for c in cfgs if c[0] in (1, 2, 4, 8)]
    else:
        keep = [c for c in cfgs if c[0] in (1, 2) and c[5] == 0]
    seen, out = set(), []
    for c in keep:
        if c[0] not in seen:
            seen.add(c[0])
            out.append(c)
    return out


# kinds: u = shared products (uniform coefficients, bitwise), x = per-tap exact,
# f = per-tap FMA chain
KINDS = (("u", 1, 1), ("x", 1, 0), ("f", 0, 0))


def _write_tu(arr, fn, tag, sh, entries):
    lines = [HEADER, '#include "ebisu_tb_launch.cuh"\n', "namespace ebisu {\n",
             f"using SH_{tag} = {sh};\n",
             f"extern const TbKernel {arr}[];\n",
             f"extern const int {arr}_n;\n",
             f"const TbKernel {arr}[] = {{\n"]
    lines += entries
    lines.append("};\n")
    lines.append(f"const int {arr}_n = {len(entries)};\n")
    lines.append("}  // namespace ebisu\n")
    _write_if_changed(os.path.join(HERE, fn), "".join(lines))


def _write_if_changed(path, text):
    """Keep the mtime of unchanged outputs (make then rebuilds only what changed)."""
    if os.path.exists(path):
        with open(path) as f:
            if f.read() == text:
                return
    with open(path, "w") as f:
        f.write(text)


def main():
    units = []
    for sid, sh, tag, cfgs in S2D:
        for kind, exact, uni in KINDS:
            arr = f"k_{tag}_{kind}"
            lst = [(t, c, 0, 0, 0, 0) for t, c in cfgs]
            if kind in ("f", "x"):
                lst = _trim_fma(lst, 2)  # per-tap kernels only serve non-uniform coefficients
            entries = [f"    EBISU_S2D_ENTRY({sid}, SH_{tag}, {t}, {c}, {NW}, {S}, {exact}, {uni}, "
                       f"double),\n"
                       for t, c, *_ in lst]
            if kind == "u" and tag in SHIFT_2D:
                # shifted-window variants first (the default per depth); the
                # rotating ones stay registered as variant 1
                entries = [f"    EBISU_S2D_ENTRY_SH({sid}, SH_{tag}, {t}, {c}, {NW}, {S}, 1, 1, "
                           f"double, {u}),\n" for t, c, u in SHIFT_2D[tag]] + entries
            if kind == "u" and tag in SHIFT_2D_AFTER:
                entries += [f"    EBISU_S2D_ENTRY_SH({sid}, SH_{tag}, {t}, {c}, {NW}, {S}, 1, 1, "
                            f"double, {u}),\n" for t, c, u in SHIFT_2D_AFTER[tag]]
            _write_tu(arr, f"ebisu_inst_{tag}_{kind}.cu", tag, sh, entries)
            units.append(arr)
    for sid, sh, tag, cfgs in S3D:
        for kind, exact, uni in KINDS:
            arr = f"k_{tag}_{kind}"
            lst = cfgs
            if kind in ("f", "x"):
                lst = _trim_fma(cfgs, 3)
            elif kind == "u":
                lst = [c for c in cfgs if c[5] == 0]
            entries = [f"    EBISU_S3D_ENTRY({sid}, SH_{tag}, {t}, {cy}, {cx}, {nwy}, {ss}, "
                       f"{dec}, {exact}, {uni}, {mb}, double),\n"
                       for t, cy, cx, nwy, ss, dec, mb in lst]
            if kind == "u" and tag in CL3D:
                entries += [f"    EBISU_S3D_CL_ENTRY({sid}, SH_{tag}, {t}, {cy}, {cx}, {nwy}, {ss}, "
                            f"1, 1),\n" for t, cy, cx, nwy, ss in CL3D[tag]]
            _write_tu(arr, f"ebisu_inst_{tag}_{kind}.cu", tag, sh, entries)
            units.append(arr)
    for sid, sh, tag, _ in S2D:
        if tag not in RA_2D:
            continue
        arr = f"k_{tag}_r"
        entries = [f"    EBISU_S2D_ENTRY_M({sid}, SH_{tag}, {t}, 4, {NW}, {ss}, 0, 1, double, {u}, {mb}),\n"
                   for t, mb, u, ss in RA_2D[tag]]
        _write_tu(arr, f"ebisu_inst_{tag}_r.cu", tag, sh, entries)
        units.append(arr)
    for sid, sh, tag, _ in H2D:
        if tag not in RA_H2D:
            continue
        arr = f"k_h2d_{tag}_r"
        entries = [f"    EBISU_H2D_ENTRY_SH({sid}, SH_{tag}, {t}, {c}, {H2D_NW}, {ss}, 0, 1, {mb}, 4),\n"
                   for t, c, mb, ss in RA_H2D[tag]]
        _write_tu(arr, f"ebisu_inst_h2d_{tag}_r.cu", tag, sh, entries)
        units.append(arr)
    for sid, sh, tag, _ in S3D:
        if tag not in RA_3D:
            continue
        arr = f"k_{tag}_r"
        entries = [f"    EBISU_S3D_ENTRY({sid}, SH_{tag}, {t}, {cy}, {cx}, {nwy}, {ss}, "
                   f"{dec}, 0, 1, {mb}, double),\n" for t, cy, cx, nwy, ss, dec, mb in RA_3D[tag]]
        _write_tu(arr, f"ebisu_inst_{tag}_r.cu", tag, sh, entries)
        units.append(arr)
    for sid, sh, tag, _ in S2D:
        arr = f"k_{tag}_s"
        entries = [f"    EBISU_S2D_ENTRY({sid}, SH_{tag}, {t}, {c}, {NW}, {S}, 1, 1, float),\n"
                   for t, c in F32_2D[tag]]
        _write_tu(arr, f"ebisu_inst_{tag}_s.cu", tag, sh, entries)
        units.append(arr)
    for sid, sh, tag, _ in S3D:
        arr = f"k_{tag}_s"
        entries = [f"    EBISU_S3D_ENTRY({sid}, SH_{tag}, {t}, {cy}, {cx}, {nwy}, {ss}, {dec}, 1, 1, "
                   f"{mb}, float),\n" for t, cy, cx, nwy, ss, dec, mb in F32_3D[tag]]
        _write_tu(arr, f"ebisu_inst_{tag}_s.cu", tag, sh, entries)
        units.append(arr)
    for sid, sh, tag, cfgs in H2D:
        star = sh.startswith("Star")
        r = int(sh.split(",")[1].strip(" >)"))
        for kind, exact, uni in (("u", 1, 1), ("x", 1, 0)):
            arr = f"k_h2d_{tag}_{kind}"
            lst = cfgs if kind == "u" else cfgs[:2]
            entries = [f"    EBISU_H2D_ENTRY({sid}, SH_{tag}, {t}, {c}, {H2D_NW}, {H2D_S}, {exact}, "
                       f"{uni}, {h2d_minb(t, r, c, star)}),\n" for t, c in lst]
            if kind == "u" and tag in SHIFT_2D:
                entries = [f"    EBISU_H2D_ENTRY_SH({sid}, SH_{tag}, {t}, {c}, {H2D_NW}, {H2D_S}, "
                           f"1, 1, {h2d_minb(t, r, c, star)}, {u}),\n"
                           for t, c, u in SHIFT_H2D[tag]] + entries
            if kind == "u" and tag in SHIFT_H2D_AFTER:
                entries += [f"    EBISU_H2D_ENTRY_SH({sid}, SH_{tag}, {t}, {c}, {H2D_NW}, {H2D_S}, "
                            f"1, 1, {h2d_minb(t, r, c, star)}, {u}),\n"
                            for t, c, u in SHIFT_H2D_AFTER[tag]]
            _write_tu(arr, f"ebisu_inst_h2d_{tag}_{kind}.cu", tag, sh, entries)
            units.append(arr)
    for sid, sh, tag, _ in H2D:
        if tag not in H2D_CLU:
            continue
        star = sh.startswith("Star")
        r = int(sh.split(",")[1].strip(" >)"))
        arr = f"k_h2d_{tag}_c"
        entries = [f"    EBISU_H2D_ENTRY_CL({sid}, SH_{tag}, {t}, {c}, {H2D_NW}, {H2D_S}, 1, 1, "
                   f"{h2d_minb(t, r, c, star)}, {u}),\n" for t, c, u in H2D_CLU[tag]]
        _write_tu(arr, f"ebisu_inst_h2d_{tag}_c.cu", tag, sh, entries)
        units.append(arr)
    reg = [HEADER, '#include <vector>\n#include <mutex>\n#include "ebisu_internal.h"\n',
           "namespace ebisu {\n"]
    for arr in units:
        reg.append(f"extern const TbKernel {arr}[];\nextern const int {arr}_n;\n")
    reg.append("const TbKernel* tb_kernels(int* count) {\n")
    reg.append("  static std::vector<TbKernel> all;\n  static std::once_flag once;\n")
    reg.append("  std::call_once(once, [] {\n")
    for arr in units:
        reg.append(f"    all.insert(all.end(), {arr}, {arr} + {arr}_n);\n")
    reg.append("  });\n  *count = (int)all.size();\n  return all.data();\n}\n")
    reg.append("}  // namespace ebisu\n")
    _write_if_changed(os.path.join(HERE, "ebisu_registry.cu"), "".join(reg))
    _write_if_changed(os.path.join(HERE, "instances.mk"),
                      "# GENERATED by gen_instances.py\nINST_SRCS := "
                      + " ".join(f"ebisu_inst_{u[2:]}.cu" for u in units) + "\n")


if __name__ == "__main__":
    main()
