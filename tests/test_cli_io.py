"""CLI + file formats (reference tests/test_io.py).  Format, parsing and gallery
enumeration checks run on CPU; the `run` / `homogenize` / batch legs need a GPU."""

import json
import struct
import subprocess
import sys

import numpy as np
import pytest

from otm_testutil import ROOT, cuda_available

from paper_2405_19991_b200.cli import EXIT_OK, EXIT_SOLVER, EXIT_USAGE, enumerate_gallery_targets, main
from paper_2405_19991_b200.homogenize import ConductivityTensor
from paper_2405_19991_b200.io import read_density, write_density

gpu = [pytest.mark.gpu, pytest.mark.skipif(not cuda_available(), reason="needs a CUDA device")]


class TestVoxelFormat:
    def test_round_trip_bit_exact(self, tmp_path):
        rho = np.random.default_rng(0).uniform(0, 1, (5, 6, 7)).astype(np.float32).astype(np.float64)
        write_density(tmp_path / "rho.otm", rho)
        back = read_density(tmp_path / "rho.otm")
        assert back.shape == (5, 6, 7) and np.array_equal(back, rho.astype(np.float32))

    def test_layout_is_little_endian_x_fastest(self, tmp_path):
        rho = np.zeros((2, 2, 2))
        rho[1, 0, 0] = 0.25
        write_density(tmp_path / "rho.otm", rho)
        raw = (tmp_path / "rho.otm").read_bytes()
        magic, nx, ny, nz = struct.unpack_from("<4sIII", raw)
        assert magic == b"OTM1" and (nx, ny, nz) == (2, 2, 2)
        vals = struct.unpack_from("<8f", raw, 16)
        assert vals[1] == 0.25 and sum(vals) == 0.25

    def test_bytes_identical_to_reference_writer(self, tmp_path):
        """Same bytes as the reference's write_density for the golden C1 final field."""
        from otm_testutil import golden
        rho = golden("traj_c1.npz")["rho_final"]
        write_density(tmp_path / "a.otm", rho)
        nx, ny, nz = rho.shape
        ref = struct.pack("<4sIII", b"OTM1", nx, ny, nz) + np.ascontiguousarray(
            rho.ravel(order="F"), dtype="<f4").tobytes()
        assert (tmp_path / "a.otm").read_bytes() == ref

    def test_corrupt_files_rejected(self, tmp_path):
        p = tmp_path / "bad.otm"
        p.write_bytes(b"NOPE" + b"\x00" * 12)
        with pytest.raises(ValueError):
            read_density(p)
        p.write_bytes(struct.pack("<4sIII", b"OTM1", 2, 2, 2) + b"\x00" * 10)
        with pytest.raises(ValueError):
            read_density(p)

    def test_out_of_range_rejected(self, tmp_path):
        with pytest.raises(ValueError):
            write_density(tmp_path / "x.otm", np.full((2, 2, 2), 1.5))


class TestGalleryEnumeration:
    def test_counts_match_published_sweep(self):
        raw, feasible = enumerate_gallery_targets([0.3, 0.2, 0.1], 0.05)
        assert len(raw) == 96 and len(feasible) == 61

    def test_component_grids(self):
        raw, _ = enumerate_gallery_targets([0.3, 0.2, 0.1], 0.05)
        assert sorted({float(t[3]) for t in raw}) == [0.0, 0.05, 0.1, 0.15, 0.2, 0.24]
        assert sorted({float(t[4]) for t in raw}) == [0.0, 0.05, 0.1, 0.14]
        assert sorted({float(t[5]) for t in raw}) == [0.0, 0.05, 0.1, 0.15]


class TestCliParsing:
    def test_usage_error_on_bad_target(self, tmp_path):
        assert main(["run", "--reso", "8", "--target", "0.3,0.2,0.1", "--out", str(tmp_path)]) == EXIT_USAGE

    def test_usage_error_on_missing_target(self, tmp_path):
        assert main(["run", "--reso", "8", "--out", str(tmp_path)]) == EXIT_USAGE

    def test_unknown_enum_exits_2(self, tmp_path):
        assert main(["run", "--reso", "8", "--target", "0.1,0.1,0.1,0,0,0", "--model", "pso",
                     "--out", str(tmp_path)]) == EXIT_USAGE

    def test_unknown_config_key_rejected(self, tmp_path):
        cfg = tmp_path / "cfg.json"
        cfg.write_text(json.dumps({"resolution": 8}))
        assert main(["run", "--config", str(cfg), "--out", str(tmp_path)]) == EXIT_USAGE

    def test_homogenize_missing_file_exits_2(self, tmp_path):
        assert main(["homogenize", "--in", str(tmp_path / "nope.otm")]) == EXIT_USAGE

    def test_gallery_dry_run(self, tmp_path, capsys):
        assert main(["gallery", "--diag", "0.3,0.2,0.1", "--step", "0.05", "--out", str(tmp_path),
                     "--dry-run"]) == EXIT_OK
        assert "96 raw combinations, 61 feasible" in capsys.readouterr().out
        assert len((tmp_path / "targets.csv").read_text().strip().splitlines()) == 62

    def test_entry_point_exists(self):
        proc = subprocess.run([sys.executable, "-m", "paper_2405_19991_b200", "--help"], capture_output=True,
                              text=True, cwd=ROOT)
        assert proc.returncode == 0 and "run" in proc.stdout and "gallery" in proc.stdout


class TestCliGpu:
    pytestmark = gpu

    def test_run_writes_all_outputs(self, tmp_path):
        out = tmp_path / "case"
        assert main(["run", "--reso", "8", "--target", "0.15,0.15,0.15,0,0,0", "--max-iter", "3", "--out",
                     str(out), "--vtk"]) == EXIT_OK
        for name in ("rho.otm", "kappa.txt", "log.csv", "manifest.json", "rho.vti"):
            assert (out / name).exists(), name
        lines = (out / "log.csv").read_text().strip().splitlines()
        assert lines[0] == "iter,g,volfrac,vstar,vcycles,ms"
        kappa = np.loadtxt(out / "kappa.txt")
        assert kappa.shape == (3, 3) and np.allclose(kappa, kappa.T)
        manifest = json.loads((out / "manifest.json").read_text())
        assert manifest["dims"] == [8, 8, 8] and manifest["penalty"] == 3.0

    def test_config_file_with_flag_override(self, tmp_path):
        cfg = tmp_path / "cfg.json"
        cfg.write_text(json.dumps({"reso": [8, 8, 8], "target": [0.15, 0.15, 0.15, 0, 0, 0], "max_iter": 2,
                                   "penalty": 2.0}))
        out = tmp_path / "run"
        assert main(["run", "--config", str(cfg), "--penalty", "4.0", "--out", str(out)]) == EXIT_OK
        manifest = json.loads((out / "manifest.json").read_text())
        assert manifest["penalty"] == 4.0 and "penalty" in manifest["overridden_flags"]
        assert manifest["max_iter"] == 2

    def test_homogenize_subcommand(self, tmp_path, capsys):
        write_density(tmp_path / "solid.otm", np.ones((8, 8, 8)))
        assert main(["homogenize", "--in", str(tmp_path / "solid.otm"), "--kappa", "1,1e-4"]) == EXIT_OK
        out = capsys.readouterr().out
        m = np.array([[float(v) for v in row.split()] for row in out.strip().splitlines()])
        assert np.abs(m - np.eye(3)).max() < 1e-5

    def test_run_deterministic_outputs(self, tmp_path):
        outs = []
        for name in ("a", "b"):
            out = tmp_path / name
            assert main(["run", "--reso", "8", "--target", "0.15,0.15,0.15,0,0,0", "--max-iter", "3", "--seed",
                         "5", "--out", str(out)]) == EXIT_OK
            outs.append((out / "rho.otm").read_bytes())
        assert outs[0] == outs[1]

    def test_solver_failure_exits_3_with_partial_outputs(self, tmp_path):
        out = tmp_path / "fail"
        assert main(["run", "--reso", "8", "--target", "0.15,0.15,0.15,0,0,0", "--tol", "1e-17", "--max-iter",
                     "3", "--out", str(out)]) == EXIT_SOLVER
        assert json.loads((out / "manifest.json").read_text())["aborted"] is True

    def test_gallery_batch_smoke(self, tmp_path):
        from paper_2405_19991_b200.cli import run_gallery
        rows = run_gallery([0.3, 0.2, 0.1], 0.05, tmp_path, reso=(8, 8, 8), jobs=1, max_iter=2)
        assert len(rows) == 61
        lines = (tmp_path / "summary.csv").read_text().strip().splitlines()
        assert len(lines) == 62 and all(l.endswith(",ok") for l in lines[1:])
        assert (tmp_path / "case_060" / "manifest.json").exists()

    def test_gallery_cases_at_once_match_one_at_a_time(self, tmp_path):
        """--per-gpu K: K cases designed concurrently from K host threads (own
        hierarchy and stream each) give the same results as one at a time."""
        from paper_2405_19991_b200.cli import run_gallery
        one = run_gallery([0.3, 0.2, 0.1], 0.1, tmp_path / "one", reso=(16, 16, 16), max_iter=6)
        four = run_gallery([0.3, 0.2, 0.1], 0.1, tmp_path / "four", reso=(16, 16, 16), max_iter=6, per_gpu=4)
        assert len(one) == len(four) > 4
        for a, b in zip(one, four):
            assert a[0] == b[0] and a[5] == b[5] == "ok"
            assert a[2] == b[2] and a[3] == b[3]          # g and volume, bit for bit


class TestReferenceBytes:
    """Every output file byte-identical to what the reference's own writers produce
    for the same result (tests/golden/io.npz, make_golden.py gen_io)."""

    def _result(self):
        from otm_testutil import golden
        import paper_2405_19991_b200 as otm
        from paper_2405_19991_b200.optimize import IterationRecord, OptimizationResult
        g = golden("io.npz")
        cfg = otm.RunConfig(dims=(5, 4, 3), target=otm.ObjectiveSpec("rel", otm.ConductivityTensor(g["target"])),
                            material=otm.MaterialParams(1.0, 1e-3, 3.5), filter=otm.FilterSpec(2.0),
                            init=otm.InitPattern("random", 0.4, seed=7), model="fixed", volume_bound=0.4,
                            oc=otm.OCParams(0.002, 0.03, 0.5), max_iter=9, symmetry="central", solver_tol=1e-7)
        log = [IterationRecord(int(i), float(gg), float(v), float(v) * 0.9, float(s), int(c), float(m))
               for i, gg, v, s, c, m in zip(g["its"], g["gs"], g["vols"], g["vst"], g["cyc"], g["ms"])]
        res = OptimizationResult(field=otm.DensityField((5, 4, 3), g["rho"], np.zeros((5, 4, 3))),
                                 kappa=otm.ConductivityTensor(g["kappa"]), log=log, converged=False, iterations=4,
                                 config=cfg)
        return g, res

    def test_write_outputs_bytes(self, tmp_path):
        from paper_2405_19991_b200.io import write_outputs
        g, res = self._result()
        written = write_outputs(res, tmp_path, vtk=True, manifest_extra={"aborted": True, "config_file": None})
        assert sorted(written) == sorted(["rho.otm", "kappa.txt", "log.csv", "manifest.json", "rho.vti"])
        for name in written:
            want = g["file_" + name.replace(".", "_")].tobytes()
            assert (tmp_path / name).read_bytes() == want, name
        assert not list(tmp_path.glob("*.tmp"))

    def test_gallery_targets_identical(self):
        from otm_testutil import golden
        g = golden("io.npz")
        for tag, diag, step in (("gallery", [0.3, 0.2, 0.1], 0.05), ("gallery2", [0.5, 0.3, 0.2], 0.04)):
            raw, feas = enumerate_gallery_targets(diag, step)
            assert np.array_equal(np.array(raw), g[f"{tag}_raw"])
            assert np.array_equal(np.array(feas), g[f"{tag}_feasible"])

    def test_config_precedence(self, tmp_path):
        """defaults < --config file < explicit flags, overridden keys reported."""
        from paper_2405_19991_b200.cli import _parser, build_run_config, merge_run_options
        cfgf = tmp_path / "c.json"
        cfgf.write_text(json.dumps({"reso": [8, 8, 16], "target": "0.2,0.2,x,0,0,0", "max-iter": 7,
                                    "kappa": [1.0, 0.001], "vtk": True}))
        args = _parser().parse_args(["run", "--config", str(cfgf), "--max-iter", "9", "--out", str(tmp_path)])
        merged, over = merge_run_options(args)
        assert merged["reso"] == (8, 8, 16) and merged["max_iter"] == 9 and merged["vtk"] is True
        assert over == ["max_iter"]
        cfg = build_run_config(merged)
        assert cfg.material.kappa_min == 0.001 and np.isnan(cfg.target.target.vec[2])
        bad = tmp_path / "bad.json"
        bad.write_text(json.dumps({"resolution": 8}))
        assert main(["run", "--config", str(bad), "--out", str(tmp_path)]) == EXIT_USAGE
