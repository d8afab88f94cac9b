// Multi-GPU run_pcv in one process: the host driver above the C ABI that shards the
// folds of a run across devices. One pcvg context per device; device i owns the contiguous fold
// range [i K / n, (i + 1) K / n) with all L chains of each fold, so per-fold statistics never cross
// devices. Every context advances on its own host thread (engine.cpp:32-61's task pool, one task per
// device); at each check interval the per-fold tables (a few doubles per fold, already on the host
// for the report) are concatenated in fold order and merged once (pcvg_merge: engine.cpp:117-253 in
// fold order, so the statistics do not depend on the device count), and the shuffle benchmark runs on
// each device's own block sums at its global stream offset with the replicate maxima MAX-combined
// (diagnostics.cpp:76-101). No chain state or block sum leaves its device. The multi-process
// equivalent over torch.distributed / NCCL is paper_2310_07002_b200/dist.py.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "../../include/pcvg.h"

struct pcvg_multi {
  std::vector<pcvg_ctx*> shards;
  std::string err;
  int K = 0, n_models = 0;
};

namespace {

struct Failure : std::runtime_error {
  int code;
  Failure(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

void chk(int32_t st, pcvg_ctx* ctx) {
  if (st != PCVG_OK) throw Failure(st, pcvg_last_error(ctx));
}

template <class F>
int32_t guarded_multi(pcvg_multi* mc, F&& f) {
  try {
    f();
    return PCVG_OK;
  } catch (const Failure& e) {
    if (mc) mc->err = e.what();
    return e.code;
  } catch (const std::exception& e) {
    if (mc) mc->err = e.what();
    return PCVG_INVALID_INPUT;
  }
}

// Runs f(i) for every shard on its own thread; rethrows the first failure (engine.cpp:32-61).
template <class F>
void for_each_shard(size_t n, F&& f) {
  std::vector<std::exception_ptr> errs(n);
  std::vector<std::thread> pool;
  for (size_t i = 0; i < n; ++i)
    pool.emplace_back([&, i] {
      try {
        f(i);
      } catch (...) {
        errs[i] = std::current_exception();
      }
    });
  for (auto& t : pool) t.join();
  for (auto& e : errs)
    if (e) std::rethrow_exception(e);
}

// Owned columns of a fold table.
struct Table {
  std::vector<double> est, lf, mc, nv, ess, rh;
  std::vector<int64_t> bt;
  std::vector<int32_t> ft, fl, rg;
  explicit Table(size_t rows = 0)
      : est(rows), lf(rows), mc(rows), nv(rows), ess(rows), rh(rows), bt(rows), ft(rows), fl(rows), rg(rows) {}
  pcvg_fold_table view() {
    return pcvg_fold_table{est.data(), lf.data(), mc.data(), nv.data(), ess.data(), rh.data(),
                           bt.data(), ft.data(), fl.data(), rg.data()};
  }
};

}  // namespace

extern "C" {

pcvg_status pcvg_multi_create(int32_t n_devices, const int32_t* devices, pcvg_multi** out) {
  return static_cast<pcvg_status>(guarded_multi(nullptr, [&] {
    if (!out || n_devices < 1 || !devices) throw Failure(PCVG_INVALID_INPUT, "need at least one device");
    auto mc = std::make_unique<pcvg_multi>();
    for (int i = 0; i < n_devices; ++i) {
      pcvg_ctx* c = nullptr;
      const int32_t st = pcvg_create(devices[i], &c);
      if (st != PCVG_OK) {
        for (pcvg_ctx* s : mc->shards) pcvg_destroy(s);
        throw Failure(st, pcvg_last_error(nullptr));
      }
      mc->shards.push_back(c);
    }
    *out = mc.release();
  }));
}

pcvg_status pcvg_multi_destroy(pcvg_multi* mc) {
  if (!mc) return PCVG_OK;
  for (pcvg_ctx* s : mc->shards) pcvg_destroy(s);
  delete mc;
  return PCVG_OK;
}

const char* pcvg_multi_last_error(const pcvg_multi* mc) { return mc ? mc->err.c_str() : ""; }

pcvg_status pcvg_multi_add_model(pcvg_multi* mc, const pcvg_dataset* data, const pcvg_folds* folds,
                                 const pcvg_model_spec* spec, const pcvg_kernel* kernel, const double* bank,
                                 int64_t bank_rows, int32_t model_id, int32_t* slot) {
  return static_cast<pcvg_status>(guarded_multi(mc, [&] {
    if (!mc || !folds) throw Failure(PCVG_INVALID_INPUT, "null argument");
    for_each_shard(mc->shards.size(), [&](size_t i) {
      int32_t s = 0;
      chk(pcvg_add_model(mc->shards[i], data, folds, spec, kernel, bank, bank_rows, model_id, &s), mc->shards[i]);
      if (i == 0 && slot) *slot = s;
    });
    mc->K = folds->K;
    ++mc->n_models;
  }));
}

pcvg_status pcvg_multi_set_kernel_policy(pcvg_multi* mc, int32_t policy) {
  return static_cast<pcvg_status>(guarded_multi(mc, [&] {
    if (!mc) throw Failure(PCVG_INVALID_INPUT, "null context");
    for (pcvg_ctx* s : mc->shards) chk(pcvg_set_kernel_policy(s, policy), s);
  }));
}

pcvg_status pcvg_multi_run(pcvg_multi* mc, const pcvg_run_config* cfg, pcvg_report* rep) {
  return static_cast<pcvg_status>(guarded_multi(mc, [&] {
    if (!mc || !cfg || !rep) throw Failure(PCVG_INVALID_INPUT, "null argument");
    if (mc->n_models < 1) throw Failure(PCVG_INVALID_INPUT, "run_pcv takes one or two models");
    if (cfg->fold_begin != 0 || cfg->fold_end != 0)
      throw Failure(PCVG_INVALID_INPUT, "pcvg_multi_run shards every fold itself");
    const int n = static_cast<int>(mc->shards.size()), K = mc->K, nm = mc->n_models, L = cfg->chains;
    if (K < n) throw Failure(PCVG_INVALID_INPUT, "more devices than folds");
    std::vector<int> fb(n), fe(n);
    for (int i = 0; i < n; ++i) {
      fb[i] = static_cast<int>(static_cast<int64_t>(i) * K / n);
      fe[i] = static_cast<int>(static_cast<int64_t>(i + 1) * K / n);
    }
    // Step 2 on every device (warm start, warm-up, centring constants)
    for_each_shard(n, [&](size_t i) {
      pcvg_run_config c = *cfg;
      c.fold_begin = fb[i];
      c.fold_end = fe[i];
      chk(pcvg_begin(mc->shards[i], &c), mc->shards[i]);
    });
    const int D = cfg->early_stop ? static_cast<int>(cfg->iters / cfg->checkpoint_every) : cfg->blocks;
    std::vector<int64_t> cks;
    if (cfg->checkpoint_every > 0)
      for (int64_t t = cfg->checkpoint_every; t < cfg->iters; t += cfg->checkpoint_every) cks.push_back(t);
    cks.push_back(cfg->iters);
    std::vector<Table> local(n);
    std::vector<std::vector<int64_t>> ldiv(n);
    std::vector<int64_t> ldrop(n), ldone(n);
    for (int i = 0; i < n; ++i) {
      local[i] = Table(static_cast<size_t>(nm) * (fe[i] - fb[i]));
      ldiv[i].resize(static_cast<size_t>(nm) * (fe[i] - fb[i]) * L);
    }
    Table full(static_cast<size_t>(nm) * K);
    std::vector<int64_t> div(static_cast<size_t>(nm) * K * L);
    rep->n_checkpoints = 0;
    int64_t done = 0;
    // global fold order, model-major (pcvg_fold_stats writes each shard model-major)
    auto gather = [&] {
      for (int i = 0; i < n; ++i) {
        const size_t nf = fe[i] - fb[i];
        for (int m = 0; m < nm; ++m) {
          const size_t src = static_cast<size_t>(m) * nf, dst = static_cast<size_t>(m) * K + fb[i];
          auto cp = [&](auto& to, const auto& from) { std::copy_n(from.begin() + src, nf, to.begin() + dst); };
          cp(full.est, local[i].est); cp(full.lf, local[i].lf); cp(full.mc, local[i].mc); cp(full.nv, local[i].nv);
          cp(full.ess, local[i].ess); cp(full.rh, local[i].rh); cp(full.bt, local[i].bt); cp(full.ft, local[i].ft);
          cp(full.fl, local[i].fl); cp(full.rg, local[i].rg);
          std::copy_n(ldiv[i].begin() + src * L, nf * L, div.begin() + dst * L);
        }
      }
    };
    // shuffle benchmark over every shard at its global offset (failed: per-fold flags or none), MAX
    auto benchmark = [&](bool with_failed, int sub_used, std::vector<double>& bmax, bool& host_path) {
      std::vector<int64_t> nonfailed(n, 0);
      for (int i = 0; i < n; ++i)
        for (int k = 0; k < fe[i] - fb[i]; ++k) nonfailed[i] += with_failed && local[i].fl[k] ? 0 : 1;
      int64_t total = 0;
      std::vector<int64_t> before(n);
      for (int i = 0; i < n; ++i) {
        before[i] = total;
        total += nonfailed[i];
      }
      std::vector<std::vector<double>> mx(n, std::vector<double>(cfg->bench_draws));
      std::vector<std::vector<int32_t>> nh(n, std::vector<int32_t>(cfg->bench_draws));
      for_each_shard(n, [&](size_t i) {
        chk(pcvg_benchmark(mc->shards[i], with_failed ? local[i].fl.data() : nullptr, before[i], total, sub_used,
                           mx[i].data(), nh[i].data()),
            mc->shards[i]);
      });
      bmax.assign(cfg->bench_draws, 0.0);
      host_path = false;
      for (int i = 0; i < n; ++i)
        for (int r = 0; r < cfg->bench_draws; ++r) {
          bmax[r] = std::max(bmax[r], mx[i][r]);
          host_path = host_path || nh[i][r] != 0;
        }
    };
    // the sequential host benchmark needs every shard's sub-block sums, in global fold order
    auto block_sums = [&](std::vector<double>& yx, std::vector<double>& yx2) {
      yx.assign(static_cast<size_t>(nm) * K * L * D, 0.0);
      yx2.assign(yx.size(), 0.0);
      for (int i = 0; i < n; ++i) {
        const size_t nf = fe[i] - fb[i], per = static_cast<size_t>(L) * D;
        std::vector<double> a(nm * nf * per), b(a.size());
        chk(pcvg_block_sums(mc->shards[i], a.data(), b.data()), mc->shards[i]);
        for (int m = 0; m < nm; ++m) {
          std::copy_n(a.begin() + m * nf * per, nf * per, yx.begin() + (static_cast<size_t>(m) * K + fb[i]) * per);
          std::copy_n(b.begin() + m * nf * per, nf * per, yx2.begin() + (static_cast<size_t>(m) * K + fb[i]) * per);
        }
      }
    };
    bool stopped = false;
    for (size_t ci = 0; ci < cks.size() && !stopped; ++ci) {
      for_each_shard(n, [&](size_t i) {
        int64_t shard_done = 0;
        chk(pcvg_advance(mc->shards[i], cks[ci] - (ci == 0 ? 0 : cks[ci - 1])), mc->shards[i]);
        pcvg_fold_table t = local[i].view();
        chk(pcvg_fold_stats(mc->shards[i], &t, ldiv[i].data(), &ldrop[i], &shard_done), mc->shards[i]);
        ldone[i] = shard_done;
      });
      done = ldone[0];
      gather();
      const bool last = ci + 1 == cks.size();
      const int sub_used = cfg->early_stop ? static_cast<int>(done / cfg->checkpoint_every) : cfg->blocks;
      bool final_ck = last;
      std::vector<double> bmax, yx, yx2;
      bool host_path = false;
      if (cfg->early_stop && !last && sub_used >= cfg->blocks) {  // the early-stop rule
        pcvg_report probe = *rep;
        std::vector<double> bench(cfg->bench_draws);
        probe.benchmark = bench.data();
        probe.snapshots = nullptr;
        probe.delta_k = nullptr;
        Table t2 = full;
        std::fill(t2.fl.begin(), t2.fl.end(), 0);
        pcvg_fold_table v2 = t2.view();
        v2.failed = nullptr;
        benchmark(false, sub_used, bmax, host_path);
        if (host_path) {
          block_sums(yx, yx2);
          chk(pcvg_merge(nm, K, cfg, done, 2, &v2, yx.data(), yx2.data(), &probe), nullptr);
        } else {
          chk(pcvg_merge_bench(nm, K, cfg, done, 2, &v2, bmax.data(), &probe), nullptr);
        }
        final_ck = probe.verdict_pass && probe.benchmark_count > 0 && std::isfinite(probe.rhat_max) &&
                   probe.mcse < probe.epistemic_se;
      }
      if (final_ck) {
        benchmark(true, sub_used, bmax, host_path);
        pcvg_fold_table v = full.view();
        if (host_path) {
          block_sums(yx, yx2);
          chk(pcvg_merge(nm, K, cfg, done, 1, &v, yx.data(), yx2.data(), rep), nullptr);
        } else {
          chk(pcvg_merge_bench(nm, K, cfg, done, 1, &v, bmax.data(), rep), nullptr);
        }
        stopped = true;
      } else {
        Table t2 = full;
        std::fill(t2.fl.begin(), t2.fl.end(), 0);
        pcvg_fold_table v2 = t2.view();
        v2.failed = nullptr;
        chk(pcvg_merge(nm, K, cfg, done, 0, &v2, nullptr, nullptr, rep), nullptr);
      }
      if (rep->snapshots) {
        double* o = rep->snapshots + 7 * ci;
        o[0] = static_cast<double>(done);
        o[1] = rep->delta_hat;
        o[2] = rep->mcse;
        o[3] = rep->epistemic_se;
        o[4] = rep->prob_a_better;
        o[5] = rep->ess_overall;
        o[6] = rep->rhat_max;
      }
      rep->n_checkpoints = static_cast<int32_t>(ci + 1);
    }
    // final per-fold tables (failed flags after exclusions were written by the merge)
    const size_t rows = static_cast<size_t>(nm) * K;
    for (size_t i = 0; i < rows; ++i) {
      rep->folds.estimate[i] = full.est[i];
      rep->folds.log_f_hat[i] = full.lf[i];
      rep->folds.mc_contribution[i] = full.mc[i];
      if (rep->folds.naive_contribution) rep->folds.naive_contribution[i] = full.nv[i];
      rep->folds.ess[i] = full.ess[i];
      rep->folds.rhat[i] = full.rh[i];
      rep->folds.batches[i] = full.bt[i];
      rep->folds.fault[i] = full.ft[i];
      if (rep->folds.dss_ridged) rep->folds.dss_ridged[i] = full.rg[i];
    }
    std::copy(div.begin(), div.end(), rep->divergences);
    rep->dropped_batch_draws = 0;
    for (int i = 0; i < n; ++i) rep->dropped_batch_draws += ldrop[i];
    rep->iters_run = done;
    // device time: the slowest device's (the devices run concurrently); kernel launches: all devices
    rep->warmup_ms = rep->sampling_ms = 0.0;
    rep->gpu_launches = 0;
    for (int i = 0; i < n; ++i) {
      double last_ms = 0.0, warm_ms = 0.0, sample_ms = 0.0;
      int64_t launches = 0;
      chk(pcvg_timing(mc->shards[i], &last_ms, &launches), mc->shards[i]);
      chk(pcvg_phase_times(mc->shards[i], &warm_ms, &sample_ms), mc->shards[i]);
      rep->gpu_launches += launches;
      rep->warmup_ms = std::max(rep->warmup_ms, warm_ms);
      rep->sampling_ms = std::max(rep->sampling_ms, sample_ms);
    }
  }));
}

}  // extern "C"
