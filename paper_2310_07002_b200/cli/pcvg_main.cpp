// pcvg - the command-line front end of the B200 PCV sampler: simulate | fit | pcv | report.
//
// A drop-in for the reference CLI (tools/pcv_main.cpp:1-279): the same subcommands, options, INI
// run configuration (config.cpp:20-120), dataset CSV (dataset.cpp:72-146), model registry
// (registry.cpp:40-96) and on-disk formats - `<stem>_bank.f64` / `_bank.json` / `_kernel.json`
// (report_io.cpp:159-222), `report.json`, `progressive.csv`, `benchmark.csv`
// (report_io.cpp:44-157) - written with the same JSON library (nlohmann/json, the reference's own
// dependency) so the files are interchangeable with the reference's readers. Every computation
// runs on the GPU through the C ABI (include/pcvg.h): Step 1 (`fit`) via pcvg_adapt_full_data,
// Steps 2-4 (`pcv`) via pcvg_run. New beside the reference: the `logistic` family and the
// `hv-block` / `hv-racine` fold schemes. Exit codes: 0 success, 2 usage or input errors, 3
// inference failures (pcv_main.cpp:259-277).
#include <charconv>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <filesystem>
#include <fstream>
#include <algorithm>
#include <iterator>
#include <map>
#include <string_view>
#include <unordered_map>
#include <memory>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include <nlohmann/json.hpp>

#include "../../include/pcvg.h"
#include "../csrc/host_common.hpp"

namespace {

using nlohmann::json;

struct UsageError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct Failure : std::runtime_error {  // status-coded library error
  int code;
  Failure(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

void check(int32_t st, pcvg_ctx* ctx = nullptr) {
  if (st != PCVG_OK) throw Failure(st, pcvg_last_error(ctx));
}

// ------------------------------------------------------------------ run settings (config.cpp grammar)
// The reference's INI dialect: `[section]` headers, `key = value` pairs, `#` starts a comment; a key
// is addressed as "section.key" (plain "key" before the first header).
std::string_view strip(std::string_view v) {
  auto blank = [](char ch) { return ch == ' ' || ch == '\t' || ch == '\r'; };
  while (!v.empty() && blank(v.front())) v.remove_prefix(1);
  while (!v.empty() && blank(v.back())) v.remove_suffix(1);
  return v;
}

class Settings {
 public:
  static Settings load(const std::string& path) {
    std::ifstream f(path, std::ios::binary);
    if (!f) throw UsageError("config file not readable: " + path);
    const std::string text((std::istreambuf_iterator<char>(f)), std::istreambuf_iterator<char>());
    return parse(text, path);
  }

  static Settings parse(std::string_view text, const std::string& origin) {
    Settings out;
    std::string prefix;
    size_t line_no = 0;
    while (!text.empty()) {
      const size_t nl = text.find('\n');
      std::string_view raw = text.substr(0, nl);
      text.remove_prefix(nl == std::string_view::npos ? text.size() : nl + 1);
      ++line_no;
      raw = strip(raw.substr(0, raw.find('#')));
      if (raw.empty()) continue;
      const std::string where = origin + ":" + std::to_string(line_no) + ": ";
      if (raw.front() == '[') {
        if (raw.back() != ']') throw UsageError(where + "section header needs a closing ']'");
        const std::string_view name = strip(raw.substr(1, raw.size() - 2));
        prefix = name.empty() ? std::string() : std::string(name) + ".";
        continue;
      }
      const size_t eq = raw.find('=');
      if (eq == std::string_view::npos) throw UsageError(where + "not a 'key = value' line");
      out.kv_[prefix + std::string(strip(raw.substr(0, eq)))] = std::string(strip(raw.substr(eq + 1)));
    }
    return out;
  }

  bool contains(const std::string& key) const { return kv_.find(key) != kv_.end(); }
  void put(const std::string& key, std::string value) { kv_[key] = std::move(value); }
  const std::string& need(const std::string& key) const {
    const auto it = kv_.find(key);
    if (it == kv_.end()) throw UsageError("setting '" + key + "' is required");
    return it->second;
  }
  std::string text(const std::string& key, const std::string& fallback) const {
    return contains(key) ? need(key) : fallback;
  }
  template <class T>
  T number(const std::string& key, T fallback) const {
    if (!contains(key)) return fallback;
    const std::string& v = need(key);
    T out{};
    const auto [end, ec] = std::from_chars(v.data(), v.data() + v.size(), out);
    if (ec != std::errc{} || end != v.data() + v.size())
      throw UsageError("setting '" + key + "' is not a number: '" + v + "'");
    return out;
  }
  long integer(const std::string& key, long fallback) const { return number<long>(key, fallback); }
  double real(const std::string& key, double fallback) const { return number<double>(key, fallback); }
  uint64_t unsigned64(const std::string& key, uint64_t fallback) const { return number<uint64_t>(key, fallback); }
  bool flag(const std::string& key, bool fallback) const {
    static const std::map<std::string, bool> kWords = {{"1", true},  {"true", true},  {"yes", true},  {"on", true},
                                                        {"0", false}, {"false", false}, {"no", false}, {"off", false}};
    if (!contains(key)) return fallback;
    const auto w = kWords.find(need(key));
    if (w == kWords.end()) throw UsageError("setting '" + key + "' must be a boolean, got '" + need(key) + "'");
    return w->second;
  }
  std::vector<std::string> items(const std::string& key) const {  // comma-separated list
    std::vector<std::string> out;
    std::string_view rest = need(key);
    if (strip(rest).empty()) return out;
    for (;;) {
      const size_t comma = rest.find(',');
      out.emplace_back(strip(rest.substr(0, comma)));
      if (comma == std::string_view::npos) break;
      rest.remove_prefix(comma + 1);
    }
    return out;
  }

 private:
  std::unordered_map<std::string, std::string> kv_;
};

// ------------------------------------------------------------------ dataset tables (dataset.cpp formats)
struct Dataset {
  std::vector<double> y, x;  // x row-major [n][n_cov]
  int n_cov = 0;
  std::vector<int32_t> group;
  std::vector<int64_t> time;
  pcvg_dataset view() const {
    return pcvg_dataset{static_cast<int64_t>(y.size()), n_cov, y.data(), x.data(),
                        group.empty() ? nullptr : group.data(), time.empty() ? nullptr : time.data()};
  }
  int n_groups() const { return group.empty() ? 0 : *std::max_element(group.begin(), group.end()) + 1; }
};

// A comma-separated table held column by column: the header names, then every field as text.
struct CsvTable {
  std::vector<std::string> names;
  std::vector<std::vector<std::string>> cols;

  static CsvTable read(const std::string& path) {
    std::ifstream f(path, std::ios::binary);
    if (!f) throw UsageError("data file not readable: " + path);
    const std::string body((std::istreambuf_iterator<char>(f)), std::istreambuf_iterator<char>());
    CsvTable t;
    std::string_view rest(body);
    size_t row = 0;
    while (!rest.empty()) {
      const size_t nl = rest.find('\n');
      std::string_view line = rest.substr(0, nl);
      rest.remove_prefix(nl == std::string_view::npos ? rest.size() : nl + 1);
      if (!line.empty() && line.back() == '\r') line.remove_suffix(1);
      if (row > 0 && line.empty()) continue;
      std::vector<std::string_view> fields;
      for (size_t from = 0;;) {
        const size_t comma = line.find(',', from);
        fields.push_back(line.substr(from, comma == std::string_view::npos ? std::string_view::npos : comma - from));
        if (comma == std::string_view::npos) break;
        from = comma + 1;
      }
      if (row == 0) {
        for (auto fv : fields) t.names.emplace_back(fv);
        t.cols.resize(t.names.size());
      } else {
        if (fields.size() != t.names.size())
          throw UsageError(path + ": line " + std::to_string(row + 1) + " has " + std::to_string(fields.size()) +
                           " fields, the header " + std::to_string(t.names.size()));
        for (size_t c = 0; c < fields.size(); ++c) t.cols[c].emplace_back(fields[c]);
      }
      ++row;
    }
    if (row == 0) throw UsageError(path + ": no header line");
    return t;
  }

  std::vector<double> numbers(const std::string& name, const std::string& path) const {
    const auto it = std::find(names.begin(), names.end(), name);
    if (it == names.end()) throw UsageError(path + ": no column named '" + name + "'");
    const auto& col = cols[static_cast<size_t>(it - names.begin())];
    std::vector<double> out(col.size());
    for (size_t r = 0; r < col.size(); ++r) {
      std::string_view v = strip(col[r]);
      const auto [end, ec] = std::from_chars(v.data(), v.data() + v.size(), out[r]);
      if (ec != std::errc{} || end != v.data() + v.size())
        throw UsageError(path + ": column '" + name + "', data row " + std::to_string(r + 1) + ": '" + col[r] +
                         "' is not a number");
    }
    return out;
  }
};

Dataset read_csv(const std::string& path, const std::string& resp, const std::vector<std::string>& covs,
                 const std::string& group, const std::string& time) {
  const CsvTable t = CsvTable::read(path);
  Dataset d;
  d.y = t.numbers(resp, path);
  if (d.y.empty()) throw UsageError(path + ": the table has no data rows");
  d.n_cov = static_cast<int>(covs.size());
  d.x.assign(d.y.size() * covs.size(), 0.0);
  for (size_t j = 0; j < covs.size(); ++j) {
    const std::vector<double> c = t.numbers(covs[j], path);
    for (size_t i = 0; i < c.size(); ++i) d.x[i * covs.size() + j] = c[i];
  }
  if (!group.empty())
    for (double v : t.numbers(group, path)) d.group.push_back(static_cast<int32_t>(std::lround(v)));
  if (!time.empty())
    for (double v : t.numbers(time, path)) d.time.push_back(std::lround(v));
  return d;
}

// Writes the dataset in the reference simulator's column order (y, covariates, group, t) with
// every real printed as %.17g (round-trip exact; registry.cpp writes the same bytes).
void write_csv(const std::string& path, const Dataset& d, const std::vector<std::string>& covs) {
  std::vector<std::string> header{"y"};
  header.insert(header.end(), covs.begin(), covs.end());
  if (!d.group.empty()) header.push_back("group");
  if (!d.time.empty()) header.push_back("t");
  std::string body;
  for (size_t h = 0; h < header.size(); ++h) body += (h ? "," : "") + header[h];
  body += '\n';
  auto real = [&](double v) {
    char buf[40];
    body.append(buf, static_cast<size_t>(std::snprintf(buf, sizeof buf, "%.17g", v)));
  };
  for (size_t i = 0; i < d.y.size(); ++i) {
    real(d.y[i]);
    for (int j = 0; j < d.n_cov; ++j) {
      body += ',';
      real(d.x[i * d.n_cov + j]);
    }
    if (!d.group.empty()) body += ',' + std::to_string(d.group[i]);
    if (!d.time.empty()) body += ',' + std::to_string(d.time[i]);
    body += '\n';
  }
  std::ofstream f(path, std::ios::binary);
  if (!f) throw UsageError("cannot create " + path);
  f << body;
}

// ------------------------------------------------------------------ registry (registry.cpp:17-96)
struct Model {
  std::string name;
  pcvg_model_spec spec{};
  std::vector<int32_t> mask;
  int dim = 0;
  std::vector<std::string> params;
};

struct Built {
  Dataset data;
  pcvg_folds folds{};
  std::vector<int32_t> test_index;
  std::vector<int64_t> intervals;
  std::vector<Model> models;
};

std::vector<std::string> param_names(const Built& b, const Model& m) {
  std::vector<std::string> n;
  const int J = b.data.n_groups();
  auto idx = [](const char* s, int i) { return std::string(s) + "[" + std::to_string(i) + "]"; };
  switch (m.spec.family) {
    case PCVG_FAMILY_GROUPED:  // grouped_regression.cpp:222-230
      for (int g = 0; g < J; ++g) n.push_back(idx("alpha", g));
      for (int p = 0; p < b.data.n_cov; ++p) n.push_back(idx("beta", p));
      n.insert(n.end(), {"mu_alpha", "log_sigma_alpha", "log_sigma_y"});
      break;
    case PCVG_FAMILY_RADON:  // radon.cpp:209-214
      for (int g = 0; g < J; ++g) n.push_back(idx("z", g));
      n.insert(n.end(), {"beta", "mu_alpha", "log_sigma_alpha2", "log_sigma_y2"});
      break;
    case PCVG_FAMILY_SEASONAL_AR:  // seasonal_ar.cpp:158-164
      for (int i = 0; i < m.spec.ar_order; ++i) n.push_back(idx("u_rho", i));
      for (int j = 0; j <= m.spec.dummies; ++j) n.push_back(idx("beta", j));
      n.push_back("log_sigma");
      break;
    case PCVG_FAMILY_RAT_GROWTH:  // rat_growth.cpp:298-308
      for (int g = 0; g < J; ++g) n.push_back(idx("alpha", g));
      if (m.spec.per_subject_slope) {
        for (int g = 0; g < J; ++g) n.push_back(idx("beta", g));
        n.insert(n.end(), {"mu_alpha", "mu_beta", "log_sigma_alpha", "log_sigma_beta", "log_sigma_y"});
      } else {
        n.insert(n.end(), {"beta", "mu_alpha", "log_sigma_alpha", "log_sigma_y"});
      }
      break;
    default:  // logistic (new family)
      n.push_back("intercept");
      for (int p = 0; p < b.data.n_cov; ++p) n.push_back(idx("beta", p));
  }
  return n;
}

Built build_models(const Settings& cfg) {
  Built b;
  std::vector<std::string> covs;
  if (cfg.contains("data.covariates")) covs = cfg.items("data.covariates");
  b.data = read_csv(cfg.need("data.path"), cfg.text("data.response", "y"), covs, cfg.text("data.group", ""),
                    cfg.text("data.time", ""));
  pcvg_dataset dv = b.data.view();
  const std::string kind = cfg.text("scheme.kind", "logo");
  const int64_t n = dv.n_obs;
  b.test_index.assign(n, 0);
  int32_t K = 0;
  if (kind == "loo") {
    check(pcvg_make_loo(n, b.test_index.data(), &K));
  } else if (kind == "logo") {
    check(pcvg_make_logo(&dv, b.test_index.data(), &K));
  } else if (kind == "kfold") {
    K = static_cast<int32_t>(std::stol(cfg.need("scheme.k")));
    check(pcvg_make_kfold(n, K, cfg.unsigned64("scheme.seed", 1), b.test_index.data()));
  } else if (kind == "time-blocks") {
    K = static_cast<int32_t>(std::stol(cfg.need("scheme.k")));
    check(pcvg_make_time_blocks(&dv, K, b.test_index.data()));
  } else if (kind == "hv-block") {  // new
    K = static_cast<int32_t>(std::stol(cfg.need("scheme.k")));
    b.intervals.assign(4 * static_cast<size_t>(K), 0);
    check(pcvg_make_hv_block(&dv, K, cfg.integer("scheme.h", 0), b.intervals.data()));
  } else if (kind == "hv-racine") {  // new
    K = static_cast<int32_t>(n);
    b.intervals.assign(4 * static_cast<size_t>(n), 0);
    check(pcvg_make_hv_racine(&dv, cfg.integer("scheme.v", 0), cfg.integer("scheme.h", 0), b.intervals.data()));
  } else {
    throw UsageError("unknown scheme.kind '" + kind + "'");
  }
  b.folds = pcvg_folds{K, b.intervals.empty() ? b.test_index.data() : nullptr,
                       b.intervals.empty() ? nullptr : b.intervals.data()};

  const std::string family = cfg.need("model.family");
  const std::string na = cfg.text("model.name_a", "M_A"), nb = cfg.text("model.name_b", "M_B");
  const bool pair = cfg.contains("model.mask_b") || cfg.contains("model.slope_b") || cfg.contains("model.floor_b") ||
                    cfg.contains("model.q_b");
  auto add = [&](const std::string& name) -> Model& {
    b.models.emplace_back();
    b.models.back().name = name;
    return b.models.back();
  };
  if (family == "grouped-reg") {
    auto mk = [&](const std::string& name, const std::string& key) {
      Model& m = add(name);
      m.spec.family = PCVG_FAMILY_GROUPED;
      if (cfg.contains(key))
        for (const auto& t : cfg.items(key)) m.mask.push_back(std::stoi(t));
    };
    mk(na, "model.mask_a");
    if (pair) mk(nb, "model.mask_b");
  } else if (family == "rat-growth") {
    auto slope = [&](const std::string& key, const std::string& fb) {
      const std::string v = cfg.text(key, fb);
      if (v == "per-subject") return 1;
      if (v == "shared") return 0;
      throw UsageError(key + " must be per-subject or shared");
    };
    add(na).spec = pcvg_model_spec{PCVG_FAMILY_RAT_GROWTH, nullptr, 1, 1, 0, 0, slope("model.slope_a", "per-subject")};
    if (pair) add(nb).spec = pcvg_model_spec{PCVG_FAMILY_RAT_GROWTH, nullptr, 1, 1, 0, 0, slope("model.slope_b", "shared")};
  } else if (family == "radon") {
    add(na).spec = pcvg_model_spec{PCVG_FAMILY_RADON, nullptr, cfg.flag("model.floor_a", true), 1, 0, 0, 0};
    if (pair) add(nb).spec = pcvg_model_spec{PCVG_FAMILY_RADON, nullptr, cfg.flag("model.floor_b", false), 1, 0, 0, 0};
  } else if (family == "seasonal-ar") {
    const int p = static_cast<int>(cfg.integer("model.p", 1));
    const std::string t = cfg.text("model.rho_transform", "half-open");
    if (t != "half-open" && t != "symmetric") throw UsageError("model.rho_transform must be half-open or symmetric");
    const int tf = t == "symmetric" ? PCVG_RHO_SYMMETRIC : PCVG_RHO_HALF_OPEN;
    add(na).spec = pcvg_model_spec{PCVG_FAMILY_SEASONAL_AR, nullptr, 1, p, static_cast<int32_t>(cfg.integer("model.q_a", 11)), tf, 0};
    if (pair) add(nb).spec = pcvg_model_spec{PCVG_FAMILY_SEASONAL_AR, nullptr, 1, p, static_cast<int32_t>(cfg.integer("model.q_b", 0)), tf, 0};
  } else if (family == "logistic") {  // new
    add(na).spec.family = PCVG_FAMILY_LOGISTIC;
  } else {
    throw UsageError("unknown model.family '" + family + "'");
  }
  for (auto& m : b.models) {
    if (!m.mask.empty()) m.spec.covariate_mask = m.mask.data();
    m.params = param_names(b, m);
    m.dim = static_cast<int>(m.params.size());
  }
  return b;
}

// ------------------------------------------------------------------ run flags (pcv_main.cpp:21-86)
struct RunFlags {
  std::string config_path, out_dir = ".";
  long seed = -1, chains = -1, iters = -1, warmup = -1, batch_size = -1, blocks = -1, bench_draws = -1;
  std::string score;
  long checkpoint_every = -1, threads = -1, device = 0, early_stop = -1;
};

int score_from_name(const std::string& s) {  // model.cpp:13-19
  if (s == "logs" || s == "LogS") return PCVG_SCORE_LOGS;
  if (s == "hs" || s == "HS") return PCVG_SCORE_HS;
  if (s == "dss" || s == "DSS") return PCVG_SCORE_DSS;
  throw UsageError("unknown score '" + s + "' (expected logs|hs|dss)");
}
const char* score_name(int s) { return s == PCVG_SCORE_HS ? "hs" : (s == PCVG_SCORE_DSS ? "dss" : "logs"); }

struct RunCfg {
  pcvg_run_config run{};
  pcvg_adapt_config fd{};
};

RunCfg make_run_config(const Settings& cfg, const RunFlags& f) {
  RunCfg r;
  pcvg_run_config& c = r.run;
  c.seed = cfg.unsigned64("run.seed", 1);
  c.chains = static_cast<int32_t>(cfg.integer("run.chains", 4));
  c.iters = cfg.integer("run.iters", 1000);
  c.warmup = cfg.integer("run.warmup", 100);
  c.batch_size = static_cast<int32_t>(cfg.integer("run.batch_size", 50));
  c.blocks = static_cast<int32_t>(cfg.integer("run.blocks", 5));
  c.bench_draws = static_cast<int32_t>(cfg.integer("run.bench_draws", 500));
  c.bench_quantile = cfg.real("run.bench_quantile", 0.99);
  c.score = score_from_name(cfg.text("run.score", "logs"));
  c.checkpoint_every = cfg.integer("run.checkpoint_every", 0);
  c.early_stop = cfg.flag("run.early_stop", false) ? 1 : 0;  // new
  r.fd.chains = static_cast<int32_t>(cfg.integer("full_data.chains", 4));
  r.fd.warmup = cfg.integer("full_data.warmup", 1000);
  r.fd.draws = cfg.integer("full_data.draws", 2000);
  r.fd.n_leapfrog = static_cast<int32_t>(cfg.integer("full_data.leapfrog", 32));
  r.fd.target_accept = cfg.real("full_data.target_accept", 0.8);
  r.fd.init_step_size = 0.0;
  if (f.seed >= 0) c.seed = static_cast<uint64_t>(f.seed);
  if (f.chains >= 0) c.chains = static_cast<int32_t>(f.chains);
  if (f.iters >= 0) c.iters = f.iters;
  if (f.warmup >= 0) c.warmup = f.warmup;
  if (f.batch_size >= 0) c.batch_size = static_cast<int32_t>(f.batch_size);
  if (f.blocks >= 0) c.blocks = static_cast<int32_t>(f.blocks);
  if (f.bench_draws >= 0) c.bench_draws = static_cast<int32_t>(f.bench_draws);
  if (!f.score.empty()) c.score = score_from_name(f.score);
  if (f.checkpoint_every >= 0) c.checkpoint_every = f.checkpoint_every;
  if (f.early_stop >= 0) c.early_stop = f.early_stop ? 1 : 0;
  return r;
}

std::string model_stem(size_t i) { return i == 0 ? "model_a" : "model_b"; }

// ------------------------------------------------------------------ JSON helpers (report_io.cpp:14-41)
json num(double v) {
  if (std::isnan(v)) return "nan";
  if (std::isinf(v)) return v > 0 ? "inf" : "-inf";
  return v;
}
json num_vec(const double* v, size_t n) {
  json a = json::array();
  for (size_t i = 0; i < n; ++i) a.push_back(num(v[i]));
  return a;
}
void csv_num(std::ofstream& out, double v) {
  if (std::isnan(v)) {
    out << "nan";
    return;
  }
  if (std::isinf(v)) {
    out << (v > 0 ? "inf" : "-inf");
    return;
  }
  char buf[32];
  std::snprintf(buf, sizeof buf, "%.17g", v);
  out << buf;
}

// ------------------------------------------------------------------ fit files (report_io.cpp:159-222)
struct Fit {
  double step_size = 0.0;
  int n_leapfrog = 32;
  std::vector<double> inv_mass, bank, rhat, ess;
  int64_t rows = 0, cols = 0, divergences = 0;
  double mean_accept = 0.0;
};

void write_fit(const std::string& dir, const std::string& stem, const Fit& f,
               const std::vector<std::string>& params) {
  const std::string base = dir + "/" + stem;
  {
    std::ofstream bank(base + "_bank.f64", std::ios::binary);
    if (!bank) throw UsageError("cannot write draw bank: " + base);
    bank.write(reinterpret_cast<const char*>(f.bank.data()),
               static_cast<std::streamsize>(f.bank.size() * sizeof(double)));
  }
  {
    json side;
    side["rows"] = static_cast<long>(f.rows);
    side["cols"] = static_cast<long>(f.cols);
    side["params"] = params;
    std::ofstream out(base + "_bank.json");
    out << side.dump(2) << '\n';
  }
  {
    json k;
    k["step_size"] = f.step_size;
    k["n_leapfrog"] = f.n_leapfrog;
    k["inv_mass_diag"] = f.inv_mass;
    k["divergences"] = static_cast<long>(f.divergences);
    k["mean_accept"] = f.mean_accept;
    k["rhat_per_param"] = num_vec(f.rhat.data(), f.rhat.size());
    k["ess_per_param"] = num_vec(f.ess.data(), f.ess.size());
    std::ofstream out(base + "_kernel.json");
    out << k.dump(2) << '\n';
  }
}

Fit read_fit(const std::string& dir, const std::string& stem) {
  const std::string base = dir + "/" + stem;
  std::ifstream side(base + "_bank.json");
  if (!side) throw UsageError("missing full-data artifacts: " + base + "_bank.json");
  const json sj = json::parse(side);
  Fit f;
  f.rows = sj.at("rows").get<long>();
  f.cols = sj.at("cols").get<long>();
  std::ifstream bank(base + "_bank.f64", std::ios::binary);
  if (!bank) throw UsageError("missing full-data artifacts: " + base + "_bank.f64");
  f.bank.resize(static_cast<size_t>(f.rows * f.cols));
  bank.read(reinterpret_cast<char*>(f.bank.data()), static_cast<std::streamsize>(f.bank.size() * sizeof(double)));
  if (!bank) throw UsageError("draw bank truncated: " + base + "_bank.f64");
  std::ifstream kin(base + "_kernel.json");
  if (!kin) throw UsageError("missing full-data artifacts: " + base + "_kernel.json");
  const json kj = json::parse(kin);
  f.step_size = kj.at("step_size").get<double>();
  f.n_leapfrog = kj.at("n_leapfrog").get<int>();
  f.inv_mass = kj.at("inv_mass_diag").get<std::vector<double>>();
  f.divergences = kj.value("divergences", 0L);
  f.mean_accept = kj.value("mean_accept", 0.0);
  return f;
}

struct Ctx {
  pcvg_ctx* h = nullptr;
  explicit Ctx(int device) { check(pcvg_create(device, &h)); }
  ~Ctx() { pcvg_destroy(h); }
};

// ------------------------------------------------------------------ subcommands
int cmd_fit(const RunFlags& flags) {
  const auto cfg = Settings::load(flags.config_path);
  const auto rc = make_run_config(cfg, flags);
  Built b = build_models(cfg);
  std::filesystem::create_directories(flags.out_dir);
  Ctx ctx(static_cast<int>(flags.device));
  const pcvg_dataset dv = b.data.view();
  for (size_t m = 0; m < b.models.size(); ++m) {
    const Model& md = b.models[m];
    Fit f;
    f.n_leapfrog = rc.fd.n_leapfrog;
    f.cols = md.dim;
    f.rows = static_cast<int64_t>(rc.fd.chains) * rc.fd.draws;
    f.inv_mass.resize(md.dim);
    f.bank.resize(static_cast<size_t>(f.rows * f.cols));
    f.rhat.resize(md.dim);
    f.ess.resize(md.dim);
    pcvg_fit out{};
    out.inv_mass_diag = f.inv_mass.data();
    out.draws = f.bank.data();
    out.rhat = f.rhat.data();
    out.ess = f.ess.data();
    check(pcvg_adapt_full_data(ctx.h, &dv, &b.folds, &md.spec, &rc.fd, rc.run.seed, static_cast<int32_t>(m), &out), ctx.h);
    f.step_size = out.step_size;
    f.divergences = out.divergences;
    f.mean_accept = out.mean_accept;
    write_fit(flags.out_dir, model_stem(m), f, md.params);
    double worst = 0.0;
    for (double r : f.rhat)
      if (std::isfinite(r)) worst = std::max(worst, r);
    std::printf("fit %-12s step_size=%.6g divergences=%ld max_param_rhat=%.4f\n", md.name.c_str(),
                f.step_size, static_cast<long>(f.divergences), worst);
  }
  return 0;
}

json report_to_json(const Built& b, const pcvg_run_config& c, int eff_b, const pcvg_report& r, int K, int L,
                    const std::vector<double>& est, const std::vector<double>& lf, const std::vector<double>& mc,
                    const std::vector<double>& ess, const std::vector<double>& rh, const std::vector<int64_t>& bt,
                    const std::vector<int32_t>& ft, const std::vector<int32_t>& fl, const std::vector<int32_t>& rg,
                    const std::vector<int64_t>& div, const std::vector<double>& dk, const std::vector<double>& snaps,
                    const std::vector<double>& bench) {
  json j;
  j["folds"] = K;
  j["chains"] = L;
  j["iters"] = static_cast<long>(c.iters);
  j["warmup"] = static_cast<long>(c.warmup);
  j["batch_size"] = eff_b;
  j["blocks"] = c.blocks;
  j["seed"] = c.seed;
  j["score"] = score_name(c.score);
  j["models"] = json::array();
  for (size_t m = 0; m < b.models.size(); ++m) {
    json jm;
    jm["name"] = b.models[m].name;
    jm["model_id"] = static_cast<int>(m);
    jm["score_total"] = num(r.score_total[m]);
    jm["numeric_faults"] = static_cast<long>(r.numeric_faults[m]);
    jm["rhat_excluded"] = r.rhat_excluded[m];
    std::vector<int> failed;
    std::vector<std::vector<long>> dv(K, std::vector<long>(L));
    json folds = json::array();
    for (int k = 0; k < K; ++k) {
      const size_t i = m * K + k;
      for (int ch = 0; ch < L; ++ch) dv[k][ch] = static_cast<long>(div[i * L + ch]);
      if (fl[i]) failed.push_back(k);
      json jf;
      jf["fold"] = k;
      jf["estimate"] = num(est[i]);
      jf["log_f_hat"] = num(lf[i]);
      jf["mc_contribution"] = num(mc[i]);
      jf["ess"] = num(ess[i]);
      jf["rhat"] = num(rh[i]);
      jf["batches"] = static_cast<long>(bt[i]);
      jf["fault"] = ft[i] != 0;
      jf["failed"] = fl[i] != 0;
      if (rg[i]) jf["dss_ridged"] = true;
      folds.push_back(jf);
    }
    jm["failed_folds"] = failed;
    jm["divergences"] = dv;
    jm["folds"] = folds;
    j["models"].push_back(jm);
  }
  j["delta_hat"] = num(r.delta_hat);
  j["delta_k"] = num_vec(dk.data(), dk.size());
  j["mcse"] = num(r.mcse);
  j["sigma2_delta"] = num(r.sigma2_delta);
  j["epistemic_se"] = num(r.epistemic_se);
  j["prob_a_better"] = num(r.prob_a_better);
  j["ess"] = num(r.ess_overall);
  j["rhat_max"] = num(r.rhat_max);
  j["dropped_batch_draws"] = static_cast<long>(r.dropped_batch_draws);
  j["benchmark"] = {{"replicates", c.bench_draws}, {"values", num_vec(bench.data(), r.benchmark_count)}};
  j["verdict"] = {{"pass", r.verdict_pass != 0},
                  {"quantile", num(r.verdict_quantile)},
                  {"quantile_value", num(r.verdict_quantile_value)},
                  {"observed", num(r.verdict_observed)}};
  json sn = json::array();
  for (int s = 0; s < r.n_checkpoints; ++s) {
    const double* o = snaps.data() + 7 * s;
    sn.push_back({{"iteration", static_cast<long>(o[0])},
                  {"delta_hat", num(o[1])},
                  {"mcse", num(o[2])},
                  {"epistemic_se", num(o[3])},
                  {"prob_a_better", num(o[4])},
                  {"ess", num(o[5])},
                  {"rhat_max", num(o[6])}});
  }
  j["snapshots"] = sn;
  return j;
}

int cmd_pcv(const RunFlags& flags) {
  const auto cfg = Settings::load(flags.config_path);
  const auto rc = make_run_config(cfg, flags);
  Built b = build_models(cfg);
  std::vector<Fit> fits;
  for (size_t m = 0; m < b.models.size(); ++m) {
    fits.push_back(read_fit(flags.out_dir, model_stem(m)));
    if (fits.back().cols != b.models[m].dim)
      throw UsageError("full-data bank of " + b.models[m].name + " has the wrong dimension");
  }
  Ctx ctx(static_cast<int>(flags.device));
  const pcvg_dataset dv = b.data.view();
  for (size_t m = 0; m < b.models.size(); ++m) {
    const pcvg_kernel kp{fits[m].step_size, fits[m].n_leapfrog, fits[m].inv_mass.data()};
    int32_t slot = 0;
    check(pcvg_add_model(ctx.h, &dv, &b.folds, &b.models[m].spec, &kp, fits[m].bank.data(), fits[m].rows,
                         static_cast<int32_t>(m), &slot), ctx.h);
  }
  const int K = b.folds.K, L = rc.run.chains, nm = static_cast<int>(b.models.size());
  const size_t rows = static_cast<size_t>(nm) * K;
  std::vector<double> est(rows), lf(rows), mc(rows), nv(rows), ess(rows), rh(rows), dk(K);
  std::vector<int64_t> bt(rows), div(rows * L);
  std::vector<int32_t> ft(rows), fl(rows), rg(rows);
  const int nck = pcvg_checkpoint_count(&rc.run);
  std::vector<double> snaps(7 * static_cast<size_t>(std::max(nck, 1))), bench(std::max(rc.run.bench_draws, 1));
  pcvg_report r{};
  r.folds = pcvg_fold_table{est.data(), lf.data(), mc.data(), nv.data(), ess.data(), rh.data(), bt.data(),
                            ft.data(), fl.data(), rg.data()};
  r.divergences = div.data();
  r.delta_k = dk.data();
  r.snapshots = snaps.data();
  r.benchmark = bench.data();
  check(pcvg_run(ctx.h, &rc.run, &r), ctx.h);
  const int eff_b = rc.run.batch_size > 0
                        ? rc.run.batch_size
                        : std::max(1, static_cast<int>(std::sqrt(static_cast<double>(rc.run.iters) * L)));
  std::filesystem::create_directories(flags.out_dir);
  {
    std::ofstream out(flags.out_dir + "/report.json");
    if (!out) throw UsageError("cannot write report: " + flags.out_dir + "/report.json");
    out << report_to_json(b, rc.run, eff_b, r, K, L, est, lf, mc, ess, rh, bt, ft, fl, rg, div, dk, snaps, bench)
               .dump(2)
        << '\n';
  }
  {
    std::ofstream out(flags.out_dir + "/progressive.csv");
    out << "iteration,delta_hat,mcse,epistemic_se,prob_a_better,ess,rhat_max\n";
    for (int s = 0; s < r.n_checkpoints; ++s) {
      const double* o = snaps.data() + 7 * s;
      out << static_cast<long>(o[0]);
      for (int c = 1; c < 7; ++c) {
        out << ',';
        csv_num(out, o[c]);
      }
      out << '\n';
    }
  }
  {
    std::ofstream out(flags.out_dir + "/benchmark.csv");
    out << "# observed_rhat_max=";
    csv_num(out, r.rhat_max);
    out << " D=" << rc.run.blocks << " R=" << rc.run.bench_draws << '\n';
    out << "replicate,rhat_max_replicate\n";
    for (int i = 0; i < r.benchmark_count; ++i) {
      out << i << ',';
      csv_num(out, bench[i]);
      out << '\n';
    }
  }
  std::printf("pcv done: delta_hat=%.6g prob_a_better=%.4f rhat_max=%.4f %s\n", r.delta_hat, r.prob_a_better,
              r.rhat_max, r.verdict_pass ? "benchmark=pass" : "benchmark=FAIL");
  std::printf("device: warm-up %.1f ms, sampling %.1f ms, %ld kernel launches, %ld iterations\n", r.warmup_ms,
              r.sampling_ms, static_cast<long>(r.gpu_launches), static_cast<long>(r.iters_run));
  return 0;
}

double json_num(const json& j) {
  if (j.is_string()) {
    const std::string s = j.get<std::string>();
    if (s == "nan") return std::nan("");
    if (s == "inf") return INFINITY;
    if (s == "-inf") return -INFINITY;
    return std::stod(s);
  }
  return j.get<double>();
}

// `pcvg report`: a summary of a report.json (ours or the reference's) - the run shape, per model the
// score total, divergences and failed folds, then the headline statistics and the benchmark verdict.
int cmd_report(const std::string& path) {
  json j;
  {
    std::ifstream in(path);
    if (!in) throw UsageError("report not readable: " + path);
    try {
      in >> j;
    } catch (const json::exception& e) {
      throw UsageError(path + " is not a valid report: " + e.what());
    }
  }
  auto fmt = [](const char* spec, double v) {
    char buf[64];
    std::snprintf(buf, sizeof buf, spec, v);
    return std::string(buf);
  };
  std::string out = "run: " + std::to_string(j.at("folds").get<long>()) + " folds x " +
                    std::to_string(j.at("chains").get<long>()) + " chains x " +
                    std::to_string(j.at("iters").get<long>()) + " iterations, score " +
                    j.at("score").get<std::string>() + "\n";
  for (const auto& m : j.at("models")) {
    long div = 0;
    for (const auto& per_fold : m.at("divergences"))
      for (const auto& c : per_fold) div += c.get<long>();
    out += "model " + m.at("name").get<std::string>() + ": score total " + fmt("%.4f", json_num(m.at("score_total"))) +
           ", " + std::to_string(div) + " divergent transitions";
    const auto& failed = m.at("failed_folds");
    if (!failed.empty()) {
      out += ", failed folds";
      for (const auto& k : failed) out += " " + std::to_string(k.get<long>());
    }
    out += "\n";
  }
  const std::pair<const char*, const char*> rows[] = {{"delta_hat", "%.4f"},    {"mcse", "%.4f"},
                                                      {"epistemic_se", "%.4f"}, {"prob_a_better", "%.4f"},
                                                      {"ess", "%.1f"},          {"rhat_max", "%.4f"}};
  for (const auto& [key, spec] : rows) out += std::string(key) + ": " + fmt(spec, json_num(j.at(key))) + "\n";
  const auto& v = j.at("verdict");
  out += "benchmark verdict: rhat_max " + fmt("%.4f", json_num(j.at("rhat_max"))) + (v.at("pass").get<bool>() ? " <= " : " > ") +
         "q" + fmt("%.2f", json_num(v.at("quantile"))) + " " + fmt("%.4f", json_num(v.at("quantile_value"))) + " (" +
         (v.at("pass").get<bool>() ? "pass" : "FAIL") + ")\n";
  std::fputs(out.c_str(), stdout);
  return 0;
}

int cmd_simulate(const std::string& family, const Settings& a, uint64_t seed, const std::string& out_dir) {
  Dataset d;
  std::vector<std::string> covs;
  pcvg::SimTruth truth;
  if (family == "grouped-reg") {  // registry.cpp:104-117
    const int J = static_cast<int>(a.integer("J", 50)), Nj = static_cast<int>(a.integer("Nj", 5)),
              P = static_cast<int>(a.integer("P", 4));
    d.n_cov = P;
    d.y.resize(static_cast<size_t>(J) * Nj);
    d.x.resize(d.y.size() * P);
    d.group.resize(d.y.size());
    pcvg::simulate_grouped(J, Nj, P, a.real("min_omitted_beta", 0.0), seed, d.y.data(), d.x.data(),
                           d.group.data(), &truth);
    for (int p = 0; p < P; ++p) covs.push_back("x" + std::to_string(p + 1));
  } else if (family == "rat-growth") {
    const int J = static_cast<int>(a.integer("J", 30));
    d.n_cov = 1;
    d.y.resize(5 * static_cast<size_t>(std::max(J, 0)));
    d.x.resize(d.y.size());
    d.group.resize(d.y.size());
    pcvg::simulate_rat(J, seed, d.y.data(), d.x.data(), d.group.data(), &truth);
    covs = {"t"};
  } else if (family == "radon") {
    const int H = static_cast<int>(a.integer("houses", 600)), C = static_cast<int>(a.integer("counties", 30));
    d.n_cov = 1;
    d.y.resize(std::max(H, 0));
    d.x.resize(d.y.size());
    d.group.resize(d.y.size());
    pcvg::simulate_radon(H, C, seed, d.y.data(), d.x.data(), d.group.data(), &truth);
    covs = {"floor"};
  } else if (family == "seasonal-ar") {
    const long T = a.integer("T", 432);
    const int p = static_cast<int>(a.integer("p", 1)), q = static_cast<int>(a.integer("q", 11));
    d.n_cov = p + q;
    const long n = std::max<long>(T - p, 0);
    d.y.resize(n);
    d.x.resize(static_cast<size_t>(n) * d.n_cov);
    d.time.resize(n);
    pcvg::simulate_seasonal(T, p, q, a.real("rho", 0.6), a.real("amp", 1.0), a.real("sigma", 1.0), seed, d.y.data(),
                            d.x.data(), d.time.data(), &truth);
    for (int i = 0; i < p; ++i) covs.push_back("lag" + std::to_string(i + 1));
    for (int j = 1; j <= q; ++j) covs.push_back("d" + std::to_string(j));
  } else {
    throw UsageError("unknown simulator family '" + family + "'");
  }
  const std::string csv = out_dir + "/" + family + ".csv";
  write_csv(csv, d, covs);
  json t;
  for (const auto& [k, v] : truth.vectors) t[k] = v;
  for (const auto& [k, v] : truth.scalars) t[k] = v;
  t["seed"] = seed;
  std::ofstream out(out_dir + "/" + family + "_truth.json");
  if (!out) throw UsageError("cannot write truth sidecar in " + out_dir);
  out << t.dump(2) << '\n';
  std::printf("wrote %s\n", csv.c_str());
  return 0;
}

// ------------------------------------------------------------------ argument parsing
const char* kUsage =
    "usage: pcvg <command> [options]\n"
    "  simulate <grouped-reg|rat-growth|radon|seasonal-ar> [--seed S] [--out DIR] [--J n] [--Nj n] [--P n]\n"
    "           [--T n] [--p n] [--q n] [--houses n] [--counties n] [--rho x] [--amp x] [--sigma x]\n"
    "           [--min-omitted-beta x]\n"
    "  fit      --config FILE [--out DIR] [run overrides]   full-data adaptation and draw bank (GPU)\n"
    "  pcv      --config FILE [--out DIR] [run overrides]   parallel cross-validation (GPU)\n"
    "  report   REPORT.json                                  summarize a report\n"
    "run overrides: --seed --chains --iters --warmup --batch-size --blocks --bench-draws --score\n"
    "               --checkpoint-every --threads --device --early-stop\n";

struct Args {
  std::vector<std::string> pos;
  std::map<std::string, std::string> opt;
};

Args parse_args(int argc, char** argv, int from) {
  Args a;
  for (int i = from; i < argc; ++i) {
    std::string s = argv[i];
    if (s == "-h" || s == "--help") throw UsageError("help");
    if (s.rfind("--", 0) == 0) {
      const auto eq = s.find('=');
      if (eq != std::string::npos) {
        a.opt[s.substr(2, eq - 2)] = s.substr(eq + 1);
      } else {
        if (i + 1 >= argc) throw UsageError("option " + s + " needs a value");
        a.opt[s.substr(2)] = argv[++i];
      }
    } else {
      a.pos.push_back(s);
    }
  }
  return a;
}

long opt_long(const Args& a, const std::string& k, long fb) {
  const auto it = a.opt.find(k);
  if (it == a.opt.end()) return fb;
  try {
    return std::stol(it->second);
  } catch (const std::exception&) {
    throw UsageError("--" + k + " expects an integer");
  }
}

RunFlags run_flags(const Args& a) {
  static const char* known[] = {"config", "out", "seed", "chains", "iters", "warmup", "batch-size", "blocks",
                                "bench-draws", "score", "checkpoint-every", "threads", "device", "early-stop"};
  for (const auto& [k, v] : a.opt) {
    bool ok = false;
    for (const char* n : known) ok = ok || k == n;
    if (!ok) throw UsageError("unknown option --" + k);
  }
  RunFlags f;
  const auto it = a.opt.find("config");
  if (it == a.opt.end()) throw UsageError("--config is required");
  f.config_path = it->second;
  if (a.opt.count("out")) f.out_dir = a.opt.at("out");
  f.seed = opt_long(a, "seed", -1);
  f.chains = opt_long(a, "chains", -1);
  f.iters = opt_long(a, "iters", -1);
  f.warmup = opt_long(a, "warmup", -1);
  f.batch_size = opt_long(a, "batch-size", -1);
  f.blocks = opt_long(a, "blocks", -1);
  f.bench_draws = opt_long(a, "bench-draws", -1);
  if (a.opt.count("score")) f.score = a.opt.at("score");
  f.checkpoint_every = opt_long(a, "checkpoint-every", -1);
  f.threads = opt_long(a, "threads", -1);  // accepted for compatibility; the device decides
  f.device = opt_long(a, "device", 0);
  f.early_stop = opt_long(a, "early-stop", -1);
  return f;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) {
    std::fputs(kUsage, stderr);
    return 2;
  }
  const std::string cmd = argv[1];
  try {
    const Args a = parse_args(argc, argv, 2);
    if (cmd == "simulate") {
      if (a.pos.size() != 1) throw UsageError("simulate needs exactly one family");
      Settings args;
      for (const auto& [k, v] : a.opt) {
        static const std::map<std::string, std::string> keys = {
            {"J", "J"}, {"Nj", "Nj"}, {"P", "P"}, {"T", "T"}, {"p", "p"}, {"q", "q"}, {"houses", "houses"},
            {"counties", "counties"}, {"rho", "rho"}, {"amp", "amp"}, {"sigma", "sigma"},
            {"min-omitted-beta", "min_omitted_beta"}};
        if (k == "seed" || k == "out") continue;
        const auto it = keys.find(k);
        if (it == keys.end()) throw UsageError("unknown option --" + k);
        args.put(it->second, v);
      }
      const std::string out = a.opt.count("out") ? a.opt.at("out") : ".";
      std::filesystem::create_directories(out);
      return cmd_simulate(a.pos[0], args, static_cast<uint64_t>(opt_long(a, "seed", 1)), out);
    }
    if (cmd == "fit") return cmd_fit(run_flags(a));
    if (cmd == "pcv") return cmd_pcv(run_flags(a));
    if (cmd == "report") {
      if (a.pos.size() != 1) throw UsageError("report needs the path of report.json");
      return cmd_report(a.pos[0]);
    }
    if (cmd == "-h" || cmd == "--help") {
      std::fputs(kUsage, stdout);
      return 0;
    }
    throw UsageError("unknown command '" + cmd + "'");
  } catch (const UsageError& e) {
    if (std::string(e.what()) == "help") {
      std::fputs(kUsage, stdout);
      return 0;
    }
    std::fprintf(stderr, "error: %s\n%s", e.what(), kUsage);
    return 2;
  } catch (const Failure& e) {
    if (e.code == PCVG_INVALID_INPUT || e.code == PCVG_UNSUPPORTED_SCORE) {
      std::fprintf(stderr, "error: %s\n", e.what());
      return 2;
    }
    std::fprintf(stderr, "inference failure: %s\n", e.what());
    return 3;
  } catch (const pcvg::Error& e) {
    std::fprintf(stderr, e.code == PCVG_INVALID_INPUT ? "error: %s\n" : "inference failure: %s\n", e.what());
    return e.code == PCVG_INVALID_INPUT ? 2 : 3;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "inference failure: %s\n", e.what());
    return 3;
  }
}
