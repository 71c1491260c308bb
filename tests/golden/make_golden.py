#!/usr/bin/env python3
"""Generate the golden fixtures that pin the CPU oracle.

Runs the UNMODIFIED reference library (compiled in place from
/root/reference/proj/src by `make -C oracle ref`, linked with the builder's
stand-in coarse solver and harness -> oracle/_ref/ref_harness) and stores its
outputs as small JSON fixtures in tests/golden/. Run in the build container
(it needs /root/reference); the fixtures are committed and travel to the GPU
box, where /root/reference does not exist.

    python tests/golden/make_golden.py
"""
from __future__ import annotations

import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
HARNESS = ROOT / "oracle" / "_ref" / "ref_harness"
OUT = Path(__file__).resolve().parent

# (file stem, harness argv)
STRUCTURE = [
    ("struct_square_2_full", ["structure", "square", "2", "neumann", "full"]),
    ("struct_square_2_dirichlet_full", ["structure", "square", "2", "dirichlet", "full"]),
    ("struct_ico_1_full", ["structure", "ico", "1", "neumann", "full"]),
    ("struct_equi_4_8_1", ["structure", "equi:4:8:1.0", "1", "neumann", "full"]),
    ("struct_grid_3_2", ["structure", "grid:3:2:2.0:1.5", "2", "neumann"]),
    ("struct_square_4", ["structure", "square", "4", "neumann"]),
    ("struct_square_4_dirichlet", ["structure", "square", "4", "dirichlet"]),
    ("struct_ico_4", ["structure", "ico", "4", "neumann"]),
    ("struct_ico_6", ["structure", "ico", "6", "neumann"]),
    ("struct_equi_4_8_3", ["structure", "equi:4:8:1.0", "3", "neumann"]),
    # SubdivisionScheme::Cubic (subdivision.cpp:116-120), "<base>+cubic"
    ("struct_square_cubic_2_full", ["structure", "square+cubic", "2", "neumann", "full"]),
    ("struct_square_cubic_3_dirichlet", ["structure", "square+cubic", "3", "dirichlet"]),
    ("struct_ico_cubic_3", ["structure", "ico+cubic", "3", "neumann"]),
    ("struct_equi_cubic_2", ["structure", "equi:4:8:1.0+cubic", "2", "neumann"]),
]
CYCLES = [
    ("cycles_square_4_dirichlet_sinsin", ["cycles", "square", "4", "dirichlet", "sinsin", "0", "12"]),
    ("cycles_square_4_uniform", ["cycles", "square", "4", "neumann", "uniform", "1", "12"]),
    ("cycles_ico_4_uniform", ["cycles", "ico", "4", "neumann", "uniform", "1", "10"]),
    ("cycles_ico_5_ylm", ["cycles", "ico", "5", "neumann", "ylm", "2", "8"]),
    ("cycles_equi_4_8_3_lr", ["cycles", "equi:4:8:1.0", "3", "neumann", "lr", "3", "10"]),
    ("cycles_ico_3_uniform_gs", ["cycles", "ico", "3", "neumann", "uniform", "4", "6", "gs"]),
    ("cycles_ico_3_uniform_sgs", ["cycles", "ico", "3", "neumann", "uniform", "4", "6", "sgs"]),
    ("cycles_ico_5_ylm_gs", ["cycles", "ico", "5", "neumann", "ylm", "2", "5", "gs"]),
    ("cycles_square_4_dirichlet_sinsin_gs", ["cycles", "square", "4", "dirichlet", "sinsin", "0", "8", "gs"]),
    ("cycles_equi_4_8_3_lr_sgs", ["cycles", "equi:4:8:1.0", "3", "neumann", "lr", "3", "6", "sgs"]),
    ("cycles_square_cubic_3_dirichlet_sinsin", ["cycles", "square+cubic", "3", "dirichlet", "sinsin", "0", "8"]),
    ("cycles_ico_cubic_3_uniform", ["cycles", "ico+cubic", "3", "neumann", "uniform", "1", "8"]),
    ("cycles_ico_cubic_2_ylm_gs", ["cycles", "ico+cubic", "2", "neumann", "ylm", "2", "5", "gs"]),
    ("cycles_ico_4_uniform_cg", ["cycles", "ico", "4", "neumann", "uniform", "1", "6", "cg"]),
    ("cycles_square_4_dirichlet_sinsin_cg", ["cycles", "square", "4", "dirichlet", "sinsin", "0", "5", "cg"]),
]
SOLVES = [
    # BASELINE configs 1-3 (config 3 takes ~30 s of reference setup)
    ("solve_config1", ["solve", "square", "4", "dirichlet", "sinsin", "0", "1e-8", "200"]),
    ("solve_config2", ["solve", "ico", "6", "neumann", "ylm", "1", "1e-8", "200"]),
    ("solve_config3", ["solve", "ico", "8", "neumann", "uniform", "1", "1e-8", "200"]),
    ("solve_equi_4_8_3_lr", ["solve", "equi:4:8:1.0", "3", "neumann", "lr", "23", "1e-10", "50"]),
    ("solve_square_6_uniform", ["solve", "square", "6", "neumann", "uniform", "5", "1e-8", "200"]),
    ("solve_config2_gs", ["solve", "ico", "6", "neumann", "ylm", "1", "1e-8", "200", "gs"]),
    ("solve_config1_sgs", ["solve", "square", "4", "dirichlet", "sinsin", "0", "1e-8", "200", "sgs"]),
    ("solve_ico_cubic_3_ylm", ["solve", "ico+cubic", "3", "neumann", "ylm", "1", "1e-8", "300"]),
    ("solve_square_cubic_4_uniform", ["solve", "square+cubic", "4", "neumann", "uniform", "5", "1e-8", "300"]),
    ("solve_config2_cg", ["solve", "ico", "6", "neumann", "ylm", "1", "1e-8", "200", "cg"]),
    # build_hierarchy's use_levels (multigrid.cpp:333-337), the paper's "as more levels are used"
    # experiment (625-vertex equilateral base, W-cycles, Gauss-Seidel), x3 here:
    # coarse solves of 9,409 / 2,401 / 625 unknowns (the stand-in's tree-sum CG above 32)
    ("solve_levels_used_2", ["solve", "equi:24:48:1.0", "3", "neumann", "uniform", "7", "1e-8", "60", "gs", "2",
                             "rediscretize", "W", "2", "2"]),
    ("solve_levels_used_3", ["solve", "equi:24:48:1.0", "3", "neumann", "uniform", "7", "1e-8", "60", "gs", "3",
                             "rediscretize", "W", "2", "2"]),
    ("solve_levels_used_all", ["solve", "equi:24:48:1.0", "3", "neumann", "uniform", "7", "1e-8", "60", "gs", "0",
                               "rediscretize", "W", "2", "2"]),
    ("solve_square_dirichlet_levels_used", ["solve", "square", "6", "dirichlet", "sinsin", "0", "1e-8", "60", "jacobi",
                                            "3"]),
    # HierarchyOptions (multigrid.hpp:99-104): Galerkin coarse operators, clamped dual areas
    # (Galerkin diverges on the flat meshes in the reference itself; the icosphere converges)
    ("solve_ico_4_galerkin", ["solve", "ico", "4", "neumann", "uniform", "5", "1e-8", "100", "gs", "0", "galerkin"]),
    ("solve_ico_5_clamp", ["solve", "ico", "5", "neumann", "uniform", "5", "1e-8", "200", "jacobi", "0", "clamp"]),
    ("solve_square_5_gs", ["solve", "square", "5", "neumann", "uniform", "5", "1e-8", "200", "gs"]),
]
PCG = [
    # gmg_preconditioned_cg (solvers.cpp:118-130): <rhs> <seed> <V|W> <pre> <post> <cycles> <tol> <maxit> [smoother]
    ("pcg_config2_v22", ["pcg", "ico", "6", "neumann", "ylm", "1", "V", "2", "2", "1", "1e-8", "100"]),
    ("pcg_ico_5_w22x2", ["pcg", "ico", "5", "neumann", "uniform", "13", "W", "2", "2", "2", "1e-9", "100"]),
    ("pcg_square_5_uniform_v11_sgs", ["pcg", "square", "5", "neumann", "uniform", "8", "V", "1", "1", "1", "1e-9",
                                      "100", "sgs"]),
    ("pcg_equi_onelevel", ["pcg", "equi:4:8:1.0", "0", "neumann", "uniform", "7", "V", "3", "3", "1", "1e-9", "30"]),
]


# write_obj / write_matrix_market (mesh_io.cpp:71-82, sparse.cpp:247-259):
# sha256 of the reference's output bytes; read_obj (mesh_io.cpp:19-69): a
# reference-written OBJ fixture and the reference's verdicts on malformed files
WRITES = [("ico", "3", "0", w) for w in ("obj", "L", "P", "R")] + [("ico", "3", "1", "L")] + \
         [("square+cubic", "2", "0", w) for w in ("obj", "L", "P", "R")] + [("equi:4:8:1.0", "2", "1", "obj")]
BAD_OBJ = {
    "vertex": "v 0 0\nf 1 2 3\n",
    "face_index": "v 0 0 0\nv 1 0 0\nv 0 1 0\nf 1 2 x\n",
    "quad": "v 0 0 0\nv 1 0 0\nv 0 1 0\nv 1 1 0\nf 1 2 3 4\n",
    "range": "v 0 0 0\nv 1 0 0\nf 1 2 3\n",
    "record": "v 0 0 0\nvn 0 0 1\n",
    "slash": "v 0 0 0\nv 1 0 0\nv 0 1 0\nf 1/1 2/2 3/3\n",
    "empty": "# nothing\n\n",
    "ok_comments": "# tri\nv 0 0 0\n\nv 1 0 0\nv 0 1 0\nf 1 2 3\n",
}


def make_io():
    import hashlib
    import tempfile
    out = {"writes": [], "bad_obj": {}}
    with tempfile.TemporaryDirectory() as td:
        for case, k, lvl, what in WRITES:
            f = Path(td) / "out"
            subprocess.run([str(HARNESS), "write", case, k, lvl, what, str(f)], check=True)
            out["writes"].append({"case": case, "k": int(k), "level": int(lvl), "what": what,
                                  "sha256": hashlib.sha256(f.read_bytes()).hexdigest()})
        for name, text in BAD_OBJ.items():
            f = Path(td) / f"{name}.obj"
            f.write_text(text)
            verdict = run(["readobj", str(f)])
            if "error" in verdict:  # paths differ between runs: keep the part after the file name
                verdict["error"] = verdict["error"].replace(str(f), "<path>")
            out["bad_obj"][name] = {"text": text, "verdict": verdict}
        obj = OUT / "ico2_ref.obj"
        subprocess.run([str(HARNESS), "write", "ico", "2", "0", "obj", str(obj)], check=True)
        out["ico2_ref_obj"] = run(["readobj", str(obj)])
    (OUT / "io.json").write_text(json.dumps(out, indent=1) + "\n")


# The downstream consumer (integrate_convection, physics.cpp:220-272): the
# reference on the CPU, oracle/_ref/convection_ref (`make -C oracle convection`).
# argv: nx ny levels t_final samples smoother cycle pre post solver [rtol=atol]
CONVECTION = [
    ("convection_32_gs_w33", ["32", "32", "3", "0.002", "3", "gs", "W", "3", "3", "gmg", "1e-7"]),
    ("convection_32_jacobi_v22", ["32", "32", "3", "0.002", "3", "jacobi", "V", "2", "2", "gmg", "1e-7"]),
    ("convection_64_sgs_f21", ["64", "32", "4", "0.001", "2", "sgs", "F", "2", "1", "gmg", "1e-6"]),
    ("convection_32_pcg", ["32", "32", "3", "0.001", "2", "gs", "W", "3", "3", "gmgpcg", "1e-7"]),
    ("convection_256_gs_w33", ["256", "256", "6", "0.00002", "2", "gs", "W", "3", "3", "gmg", "1e-6"]),
]


def make_convection(only):
    exe = ROOT / "oracle" / "_ref" / "convection_ref"
    if not exe.exists():
        subprocess.run(["make", "-C", str(ROOT / "oracle"), "convection", "-j8"], check=True)
    for stem, argv in CONVECTION:
        if only and stem not in only:
            continue
        res = subprocess.run([str(exe), *argv], check=True, capture_output=True, text=True)
        data = json.loads(res.stdout)
        data["_argv"] = argv
        (OUT / f"{stem}.json").write_text(json.dumps(data, separators=(",", ":")) + "\n")
        print(stem, file=sys.stderr)


def run(argv):
    res = subprocess.run([str(HARNESS), *argv], check=True, capture_output=True, text=True)
    return json.loads(res.stdout)


def main() -> int:
    if not HARNESS.exists():
        subprocess.run(["make", "-C", str(ROOT / "oracle"), "ref", "-j8"], check=True)
    only = set(sys.argv[1:])  # optional: regenerate just these stems
    if not only or "io" in only:
        make_io()
    make_convection(only)
    for stem, argv in STRUCTURE + CYCLES + SOLVES + PCG:
        if only and stem not in only:
            continue
        data = run(argv)
        data["_argv"] = argv
        (OUT / f"{stem}.json").write_text(json.dumps(data, separators=(",", ":")) + "\n")
        print(stem, file=sys.stderr)
    return 0


if __name__ == "__main__":
    sys.exit(main())
