"""The `pcvg` command-line front end (paper_2310_07002_b200/cli/pcvg_main.cpp) against the
reference's own file formats (tools/pcv_main.cpp, registry.cpp:98-165, report_io.cpp):
* CPU: `pcvg simulate` writes the same CSV and truth sidecar bytes as the reference's
  run_simulator; usage errors exit 2; `pcvg report` summarises a reference report.json;
* GPU: `pcvg fit` writes a bank the reference's read_full_data_fit loads, and `pcvg pcv` writes
  report.json / progressive.csv / benchmark.csv with the reference's structure and values within
  Monte Carlo error of the reference engine on the same bank."""
import ctypes as C
import json
import os
import subprocess

import numpy as np
import pytest

import _oracle as O
from paper_2310_07002_b200 import abi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "paper_2310_07002_b200", "lib", "pcvg")

pytestmark = pytest.mark.skipif(not os.path.exists(CLI), reason="pcvg CLI not built")


def run(*args, cwd=None):
    return subprocess.run([CLI, *args], capture_output=True, text=True, cwd=cwd, timeout=600)


SIMS = [("grouped-reg", ["--J", "12", "--Nj", "4", "--P", "3"], "J=12;Nj=4;P=3"),
        ("rat-growth", ["--J", "9"], "J=9"),
        ("radon", ["--houses", "90", "--counties", "9"], "houses=90;counties=9"),
        ("seasonal-ar", ["--T", "120", "--p", "2", "--q", "11"], "T=120;p=2;q=11")]


@pytest.mark.ref
@pytest.mark.parametrize("family,args,ref_args", SIMS)
def test_simulate_matches_reference_files(tmp_path, family, args, ref_args):
    ours, theirs = tmp_path / "ours", tmp_path / "ref"
    ours.mkdir()
    theirs.mkdir()
    r = run("simulate", family, "--seed", "7", "--out", str(ours), *args)
    assert r.returncode == 0, r.stderr
    lib = O.ref()
    lib.pcvref_run_simulator.argtypes = [C.c_char_p, C.c_char_p, C.c_uint64, C.c_char_p]
    assert lib.pcvref_run_simulator(family.encode(), ref_args.encode(), 7, str(theirs).encode()) == 0
    for name in (f"{family}.csv", f"{family}_truth.json"):
        assert (ours / name).read_bytes() == (theirs / name).read_bytes(), name


def test_usage_errors_exit_2(tmp_path):
    assert run().returncode == 2
    assert run("bogus").returncode == 2
    assert run("fit").returncode == 2  # --config is required
    assert run("pcv", "--config", str(tmp_path / "missing.cfg")).returncode == 2
    assert run("simulate", "nope").returncode == 2
    assert run("--help").returncode == 0


def write_config(tmp_path, csv, extra=""):
    cfg = tmp_path / "run.cfg"
    cfg.write_text(f"""# grouped regression, leave-one-group-out (paper Ex-1 style)
[data]
path = {csv}
covariates = x1, x2, x3
group = group
[scheme]
kind = logo
[model]
family = grouped-reg
mask_a = 1, 1, 1
mask_b = 1, 1, 0
[run]
seed = 3
chains = 4
iters = 120
warmup = 20
batch_size = 10
bench_draws = 40
checkpoint_every = 60
[full_data]
chains = 4
warmup = 400
draws = 200
{extra}""")
    return cfg


@pytest.mark.gpu
def test_fit_and_pcv_write_reference_formats(tmp_path):
    assert run("simulate", "grouped-reg", "--seed", "5", "--out", str(tmp_path), "--J", "20", "--Nj", "5",
               "--P", "3", "--min-omitted-beta", "1.0").returncode == 0
    cfg = write_config(tmp_path, tmp_path / "grouped-reg.csv")
    out = tmp_path / "out"
    r = run("fit", "--config", str(cfg), "--out", str(out))
    assert r.returncode == 0, r.stderr
    assert r.stdout.startswith("fit M_A")
    for stem in ("model_a", "model_b"):
        side = json.loads((out / f"{stem}_bank.json").read_text())
        assert side["rows"] == 800 and side["cols"] == len(side["params"])
        kern = json.loads((out / f"{stem}_kernel.json").read_text())
        assert kern["step_size"] > 0 and len(kern["inv_mass_diag"]) == side["cols"]
        bank = np.fromfile(out / f"{stem}_bank.f64")
        assert bank.size == side["rows"] * side["cols"] and np.all(np.isfinite(bank))
        if O.have_ref():  # the reference's own reader loads our files
            lib = O.ref()
            lib.pcvref_read_fit.argtypes = [C.c_char_p, C.c_char_p, abi.P_i64, abi.P_i64, abi.P_f64, abi.P_f64]
            rows, cols, step = C.c_int64(), C.c_int64(), C.c_double()
            first = np.zeros(side["cols"])
            assert lib.pcvref_read_fit(str(out).encode(), stem.encode(), C.byref(rows), C.byref(cols),
                                       C.byref(step), abi.ptr(first, C.c_double)) == 0
            assert rows.value == 800 and step.value == kern["step_size"]
            np.testing.assert_array_equal(first, bank[:side["cols"]])
    r = run("pcv", "--config", str(cfg), "--out", str(out))
    assert r.returncode == 0, r.stderr
    assert r.stdout.startswith("pcv done: delta_hat=")
    rep = json.loads((out / "report.json").read_text())
    for key in ("folds", "chains", "iters", "warmup", "batch_size", "blocks", "seed", "score", "models",
                "delta_hat", "delta_k", "mcse", "sigma2_delta", "epistemic_se", "prob_a_better", "ess",
                "rhat_max", "dropped_batch_draws", "benchmark", "verdict", "snapshots"):
        assert key in rep, key
    assert rep["folds"] == 20 and rep["chains"] == 4 and rep["score"] == "logs"
    assert [m["name"] for m in rep["models"]] == ["M_A", "M_B"]
    m0 = rep["models"][0]
    assert len(m0["folds"]) == 20 and len(m0["divergences"]) == 20 and len(m0["divergences"][0]) == 4
    assert set(m0["folds"][0]) >= {"fold", "estimate", "log_f_hat", "mc_contribution", "ess", "rhat",
                                   "batches", "fault", "failed"}
    assert len(rep["snapshots"]) == 2 and rep["snapshots"][-1]["iteration"] == 120
    assert rep["benchmark"]["replicates"] == 40 and len(rep["benchmark"]["values"]) == 40
    prog = (out / "progressive.csv").read_text().splitlines()
    assert prog[0] == "iteration,delta_hat,mcse,epistemic_se,prob_a_better,ess,rhat_max" and len(prog) == 3
    bench = (out / "benchmark.csv").read_text().splitlines()
    assert bench[0].startswith("# observed_rhat_max=") and bench[0].endswith("D=5 R=40")
    assert bench[1] == "replicate,rhat_max_replicate" and len(bench) == 42
    r = run("report", str(out / "report.json"))
    assert r.returncode == 0 and "delta_hat:" in r.stdout
    if O.have_ref():  # the reference engine + writers on the same data, folds and banks
        from paper_2310_07002_b200 import pcv
        import csv as _csv
        rows = list(_csv.reader(open(tmp_path / "grouped-reg.csv")))[1:]
        arr = np.array(rows, dtype=float)
        d = abi.DatasetArrays(arr[:, 0], arr[:, 1:4], arr[:, 4].astype(np.int32))
        f = pcv.make_logo_scheme(d)
        fa = f.arrays()
        models, kernels, banks = [], [], []
        for stem, mask in (("model_a", [1, 1, 1]), ("model_b", [1, 1, 0])):
            models.append(O.RModel(d, fa, abi.SpecArrays(abi.FAMILY_GROUPED, covariate_mask=mask)))
            kern = json.loads((out / f"{stem}_kernel.json").read_text())
            kernels.append(abi.KernelArrays(kern["step_size"], kern["n_leapfrog"], kern["inv_mass_diag"]))
            banks.append(np.fromfile(out / f"{stem}_bank.f64").reshape(800, -1))
        cfgr = abi.run_config(chains=4, iters=120, warmup=20, batch_size=10, bench_draws=40, checkpoint_every=60,
                              seed=3)
        refdir = tmp_path / "ref"
        refdir.mkdir()
        arr_h, ks, bptr, brows, ids, keep = O._run(None, [m.h for m in models], [0, 1], kernels, banks, cfgr, 0)
        lib = O.ref()
        lib.pcvref_run_pcv_files.argtypes = [C.c_int32, C.POINTER(C.c_void_p), abi.P_i32, C.POINTER(abi.Kernel),
                                             C.POINTER(abi.P_f64), abi.P_i64, C.POINTER(abi.RunConfig), C.c_int32,
                                             C.c_char_p]
        assert lib.pcvref_run_pcv_files(2, arr_h, abi.ptr(ids, C.c_int32), ks, bptr, abi.ptr(brows, C.c_int64),
                                        C.byref(cfgr), 0, str(refdir).encode()) == 0
        ref = json.loads((refdir / "report.json").read_text())
        assert set(ref) == set(rep)
        assert set(ref["models"][0]) == set(m0)
        assert set(ref["models"][0]["folds"][0]) == set(m0["folds"][0])
        assert set(ref["verdict"]) == set(rep["verdict"]) and set(ref["snapshots"][0]) == set(rep["snapshots"][0])
        for k in ("folds", "chains", "iters", "warmup", "batch_size", "blocks", "seed", "score"):
            assert ref[k] == rep[k], k
        tol = 4.0 * np.hypot(rep["mcse"], ref["mcse"]) + 1e-9
        assert abs(rep["delta_hat"] - ref["delta_hat"]) <= tol, (rep["delta_hat"], ref["delta_hat"], tol)
        assert (refdir / "progressive.csv").read_text().splitlines()[0] == prog[0]
        assert (refdir / "benchmark.csv").read_text().splitlines()[1] == bench[1]
