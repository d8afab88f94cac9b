#!/usr/bin/env python
"""PCV sampler benchmark (BASELINE.json metric: chain-steps/sec).

Workload (BASELINE.json configs[1], the single-GPU config the metric is quoted on): Bernoulli-logit
regression, synthetic N=10,000 observations x P=50 covariates (+ intercept), LOO CV = 10,000 folds
x 8 chains = 80,000 HMC chains, n_leapfrog = 32, FP64. One "step" = one HMC transition of every
chain + its log_pred + the online accumulator update (engine.cpp:360-373). Kernel parameters and
the warm-start draw bank are the reference's own adapt_full_data output on this dataset
(tests/golden/cfg2_logistic_bench.npz). Multi-GPU: folds are sharded across ranks (strong
scaling, total work fixed); no collective on the data path, the per-fold statistics are gathered
once after the timed region. The line also carries `time_to_converged`: the wall-clock of one
run_pcv call with the early-stop rule on cfg4 (BASELINE configs[3], the early-stopping config).

  python bench.py [--gpus N --steps K --warmup W] [--impl reference]
  torchrun --nproc-per-node N bench.py --gpus N ...
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))

N_OBS, P, L, N_LF = 10000, 50, 8, 32
WORKLOAD = "cfg2: logistic regression N=10000 P=50, LOO 10000 folds x 8 chains, n_leapfrog=32, FP64"
# Algorithmic FLOPs of one chain-step: n_lf gradient passes, each two
# N x (P+1) contractions (X.theta and X^T.r) = 4 N (P+1) flop; log density fused, transcendentals
# not counted.
FLOP_PER_CHAIN_STEP = N_LF * 4.0 * N_OBS * (P + 1)
CPU_SAMPLE_FOLDS = 64


def peak_tf32():
    """Dense TF32 tensor peak: half the measured dense bf16 figure (tcgen05 kind::tf32 runs at half
    the kind::f16 rate)."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)["bf16_tflops"] / 2.0, "MEASURED_PEAKS.json bf16_tflops / 2 (dense TF32)"
    except (OSError, KeyError, ValueError):
        return 1125.0, "nominal dense TF32 (2.25 PF/s bf16 / 2; MEASURED_PEAKS.json absent)"


def peak_fp64():
    path = os.path.join(ROOT, "profiles", "r01_fp64_peaks.json")
    with open(path) as f:
        pk = json.load(f)
    return pk["dmma_tflops_bps8"], "measured FP64 DMMA peak (profiles/r01_fp64_peaks.json; "\
        "MEASURED_PEAKS.json has no FP64 figure)"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index),
                 "--query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([c.strip() for c in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            self.proc.wait()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if len(r) > 4 + i and r[4 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons, "samples": len(self.rows)}


def load_inputs():
    from make_golden import load
    d, f, models, _ = load("cfg2_logistic_bench")
    kw, kp, bank = models[0]
    return d, f, kp, bank


def workload_config(folds, world):
    """The `config` block shared by both arms (the reference arm times a fold sample of the same
    workload; the sample is stated in its cpu_baseline)."""
    return {"workload": WORKLOAD, "folds": folds, "chains_per_fold": L, "n_obs": N_OBS, "covariates": P,
            "n_leapfrog": N_LF, "chains": folds * L,
            "l2": "flushed between timed steps (256 MiB memset); X (4 MB) then re-read from HBM",
            "parallelism": f"fold-sharded x{world}"}


def cpu_sample(folds_total, steps, warmup, threads, prefer_ref=True):
    """The reference's own Step 2-3 task loop on a bounded fold sample (oracle/_ref, through
    oracle/refarm.py, which never loads the product library), or the C port when the reference
    build is absent. Returns (chain-steps/s, kind, sample description)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import refarm
    return refarm.cpu_sample(folds_total, CPU_SAMPLE_FOLDS, L, steps, warmup, threads, prefer_ref)


def run_reference(args, rank, world):
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    value, kind, sample = cpu_sample(N_OBS, args.steps, args.warmup, threads)
    line = {"impl": "reference", "metric": "chain-steps/sec", "value": value, "unit": "chain-steps/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * N_OBS * L / value, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_config(args.folds or N_OBS, args.gpus),
            "cpu_baseline": {"value": value, "unit": "chain-steps/s", "cores": threads, "kind": kind,
                             "sample": sample},
            "e2e": {"value": value, "unit": "chain-steps/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


CONVERGE_WORKLOADS = {
    "cfg2k": ("cfg2 K-fold: logistic N=10000 P=50, K=10 (seed 1) x 8 chains (BASELINE configs[1], the bench "
              "data and fit), check every 50 iterations, at most 2000"),
    "cfg4": ("cfg4: seasonal AR(2)+11 dummies T=5000, hv-block K=100 h=12 (BASELINE configs[3], the "
             "early-stopping configuration), M_A + M_B x 4 chains, check every 50 iterations, at most 2000"),
}


def time_to_converged(world, local, dist, which="cfg2k"):
    """Wall-clock to R-hat-converged elpd (the second half of BASELINE.json's metric) through the
    public API with host inputs: run_pcv with the early-stop rule, one call (one GPU)
    or the fold-sharded driver (N ranks), max over ranks. cfg2 K-fold is the bench's own data, fit
    and chain count per fold (its LOO scheme needs ~6,000 iterations); cfg4 is the
    hv-block configuration of BASELINE configs[3]."""
    from make_golden import load
    from paper_2310_07002_b200 import pcv
    if which == "cfg2k":
        d, _, models, _ = load("cfg2_logistic_bench")
        folds = pcv.make_kfold_scheme(d, 10, 1)
        kp, bank = models[0][1], models[0][2]
        inputs = [pcv.ModelInput(pcv.LogisticModel("M_A", d, folds), pcv.FullDataFit(kp, bank), 0)]
        L, chains = 8, 10 * 8
    else:
        d, f, models, _ = load("cfg4_seasonal_bench")
        inputs = [pcv.ModelInput(pcv.SeasonalARModel(f"M{i}", d, f, kw["ar_order"], kw["dummies"], kw["rho_transform"]),
                                 pcv.FullDataFit(kp, bank), i) for i, (kw, kp, bank) in enumerate(models)]
        L, chains = 4, 800
    cfg = pcv.RunConfig(chains=L, iters=2000, warmup=100, batch_size=50, blocks=5, bench_draws=500, seed=1,
                        checkpoint_every=50, early_stop=1)
    if dist:
        dist.barrier()
    t0 = time.perf_counter()
    if dist:
        from paper_2310_07002_b200 import dist as pdist
        rep = pdist.run_pcv_sharded(inputs, cfg, device=local)
    else:
        rep = pcv.run_pcv(inputs, cfg, device=local)
    wall = time.perf_counter() - t0
    if dist:
        import torch
        t = torch.tensor([wall], dtype=torch.float64, device="cuda" if dist.get_backend() == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        wall = float(t.item())
    return {"workload": CONVERGE_WORKLOADS[which], "iters_run": int(rep["iters_run"]),
            "stopped_early": bool(rep["iters_run"] < cfg.iters), "wall_s": wall,
            "device_s": (rep["warmup_ms"] + rep["sampling_ms"]) / 1e3 if not dist else None,
            "rhat_max": rep["rhat_max"], "verdict_quantile_value": rep["verdict_quantile_value"],
            "delta_hat": rep["delta_hat"], "mcse": rep["mcse"], "epistemic_se": rep["epistemic_se"],
            "chain_steps": chains * (int(rep["iters_run"]) + cfg.warmup),
            "note": "one pcv.run_pcv call with host inputs (upload, warm start, warm-up, sampling with the rule "
                    "at every check interval, report); the wall-clock includes the context's creation"}


def relaunch_ranks(n):
    """`bench.py --gpus N` outside torchrun: start the N ranks (one per GPU) ourselves."""
    import socket
    import torch
    have = torch.cuda.device_count()
    if have < n and "PCVG_FORCE_DEVICE" not in os.environ:
        print(f"bench.py: --gpus {n} needs {n} visible GPUs, found {have}", file=sys.stderr)
        sys.exit(2)
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    sys.exit(subprocess.call(cmd))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-converge", action="store_true", help="skip the time-to-R-hat-converged leg (cfg4)")
    ap.add_argument("--folds", type=int, default=0, help="debug: limit the fold count")
    ap.add_argument("--fp32", action="store_true",
                    help="the separately reported FP32 variant (glm32_kernel: tcgen05 kind::tf32, "
                         "hi/lo split operands); device-timed only")
    args = ap.parse_args()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if "PCVG_FORCE_DEVICE" in os.environ:  # N ranks sharing one GPU (test of the multi-rank path)
        local = int(os.environ["PCVG_FORCE_DEVICE"])
    if args.impl == "reference":
        return run_reference(args, rank, world)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        relaunch_ranks(args.gpus)
    if world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr)
        sys.exit(2)

    import torch
    from paper_2310_07002_b200 import abi, pcv
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        # NCCL over NVLink between the GPUs; PCVG_DIST_BACKEND=gloo runs the same multi-rank logic
        # with host collectives (used to exercise N ranks on one GPU: no kernel waits on another)
        backend = os.environ.get("PCVG_DIST_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    d, f, kp, bank = load_inputs()
    K = args.folds or f.K
    from paper_2310_07002_b200.dist import shard_range
    fb, fe = shard_range(K, rank, world)
    model = pcv.LogisticModel("M_A", d, f)
    cfg = pcv.RunConfig(chains=L, iters=args.steps, warmup=args.warmup, batch_size=min(50, args.steps),
                        blocks=5, bench_draws=100, seed=1, fold_begin=fb, fold_end=fe)
    ctx = pcv.Context(local)
    if args.fp32:
        ctx.set_kernel_policy(ctx.KERNEL_TF32)
        args.no_e2e = args.no_cpu = args.no_converge = True
    ctx.add_model(model, kp, bank, model_id=0)
    ctx.begin(cfg)  # Step 2: warm start + args.warmup untimed warm-up transitions
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    _, launches0 = ctx.last_advance_ms()
    step_ms = []
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            flush.zero_()  # evict L2 (126 MB) between timed steps
            torch.cuda.synchronize()
            if dist:
                dist.barrier()
            ctx.advance(1)  # one HMC transition of every chain; CUDA events inside libpcvg
            step_ms.append(ctx.last_advance_ms()[0])
    _, launches1 = ctx.last_advance_ms()
    local_ms = float(np.sum(step_ms))
    if dist:
        t = torch.tensor([local_ms], device="cuda" if dist.get_backend() == "nccl" else "cpu", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    else:
        total_ms = local_ms
    chains_total = K * L
    value = chains_total * args.steps / (total_ms / 1e3)
    # per-fold statistics of this shard -> rank 0 -> Step-4 merge (untimed)
    cols, divs, dropped, done = ctx.fold_stats(fe - fb)
    if dist:
        from paper_2310_07002_b200 import dist as pdist
        cols = pdist.gather_fold_tables(cols, 1)
    result = None
    if rank == 0:
        rep = pcv.merge(1, K, cfg, done, 0, cols)
        result = {"score_total_elpd": rep["delta_hat"], "mcse": rep["mcse"],
                  "epistemic_se": rep["epistemic_se"], "rhat_max": rep["rhat_max"],
                  "ess_overall": rep["ess_overall"], "iters": int(done)}
    ctx.close()

    # roofline of the dominant kernel (glm_kernel<logistic,52>: one launch per step)
    peak, peak_src = peak_fp64() if not args.fp32 else peak_tf32()
    per_launch_ms = local_ms / args.steps
    achieved = FLOP_PER_CHAIN_STEP * (fe - fb) * L / (per_launch_ms * 1e-3) / 1e12
    traffic = None
    prof = os.path.join(ROOT, "profiles", "r02_ncu_glm.json")  # ncu --set full of the current kernel
    if os.path.exists(prof):
        with open(prof) as fh:
            pj = json.load(fh)
            traffic = pj.get("dram_bytes_per_launch") or pj.get("launches", [{}])[0].get("dram_bytes_per_launch")
    line = None
    if rank == 0:
        line = {"metric": "chain-steps/sec", "value": value, "unit": "chain-steps/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": total_ms / args.steps,
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
                "dtype": "f32 (tf32 hi/lo split; chain state f64)" if args.fp32 else "f64",
                "data": "synthetic",
                "config": workload_config(K, world),
                "roofline": {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                             "frac": achieved / peak, "traffic": traffic,
                             "flop_per_chain_step": FLOP_PER_CHAIN_STEP, "peak_source": peak_src,
                             "kernel": "glm32_kernel (tcgen05 kind::tf32)" if args.fp32 else "glm_kernel<logistic,52> (FP64 DMMA)",
                             "traffic_source": "profiles/r02_ncu_glm.json (ncu --set full of the full-wave "
                                               "sampling launch, dram read+write)"},
                "clocks": clk.summary(), "gpu_launches": int(launches1 - launches0), "result": result}
    # e2e: the public API call with host buffers (pcvg_run: H2D of data/bank, Step 2 + Step 3,
    # per-fold + Step-4 statistics, D2H of the report), wall-clock, max over ranks.
    if not args.no_e2e:
        t0 = time.perf_counter()
        phases = None
        close_s = 0.0
        if world == 1:  # pcv.run_pcv's steps; the clock stops when the report is on the host
            c2 = pcv.Context(local)
            t1 = time.perf_counter()
            c2.add_model(model, kp, bank, model_id=0)
            t2 = time.perf_counter()
            rep = c2.run(pcv.RunConfig(chains=L, iters=args.steps, warmup=args.warmup,
                                       batch_size=min(50, args.steps), blocks=5, bench_draws=100, seed=1))
            t3 = time.perf_counter()
            c2.close()  # context teardown (device buffers back to the stream-ordered pool): timed
            t4 = time.perf_counter()
            phases = {"context_s": t1 - t0, "add_model_s": t2 - t1, "run_s": t3 - t2,
                      "run_device_sampler_s": (rep["warmup_ms"] + rep["sampling_ms"]) / 1e3,
                      "teardown_s": t4 - t3}
            d2h = sum(v.nbytes for v in rep.values() if isinstance(v, np.ndarray))
        else:  # the fold-sharded multi-GPU driver (dist.run_pcv_sharded): tables gathered, device
            # shuffle benchmark at global stream offsets, MAX-reduced
            from paper_2310_07002_b200 import dist as pdist
            rep = pdist.run_pcv_sharded([pcv.ModelInput(model, pcv.FullDataFit(kp, bank), 0)],
                                        pcv.RunConfig(chains=L, iters=args.steps, warmup=args.warmup,
                                                      batch_size=min(50, args.steps), blocks=5,
                                                      bench_draws=100, seed=1), device=local)
            d2h = sum(v.nbytes for v in rep.values() if isinstance(v, np.ndarray))
        torch.cuda.synchronize()
        e2e_s = time.perf_counter() - t0
        if dist:
            t = torch.tensor([e2e_s], device="cuda" if dist.get_backend() == "nccl" else "cpu", dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_s = float(t.item())
        h2d = d.y.nbytes + d.x.nbytes + f.test_index.nbytes + bank.nbytes + kp.inv_mass_diag.nbytes
        if line is not None:
            steps_all = args.steps + args.warmup
            line["e2e"] = {"value": chains_total * steps_all / e2e_s, "unit": "chain-steps/s",
                           "h2d_bytes_per_step": int(h2d / steps_all), "d2h_bytes_per_step": int(d2h / steps_all),
                           "wall_s": e2e_s, "chain_steps": chains_total * steps_all, "phases": phases,
                           "note": "run_pcv (1 GPU: context, add_model, pcvg_run; N GPUs: dist.run_pcv_sharded) "
                                   "with host inputs: upload, warm start, warm-up + sampling, per-fold stats, "
                                   "shuffle benchmark (R=100, on device), report download and context "
                                   "teardown"}
    if not args.no_converge:
        conv = time_to_converged(world, local, dist, "cfg2k")
        conv4 = time_to_converged(world, local, dist, "cfg4")
        if line is not None:
            line["time_to_converged"] = conv
            line["time_to_converged_cfg4"] = conv4
    if line is not None and world == 1 and not args.no_cpu:
        threads = os.cpu_count() or 1
        cv, kind, sample = cpu_sample(K, 12, 1, threads)
        line["cpu_baseline"] = {"value": cv, "unit": "chain-steps/s", "cores": threads, "kind": kind,
                                "sample": sample}
    if line is not None:
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
