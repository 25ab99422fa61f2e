// memplan command-line front end: gen-trace, pack, plan, estimate, simulate,
// validate, sweep, list-presets.
//
// Verb semantics and outputs follow the reference CLI (proj/src/cli.cpp:59-623);
// the argument parser is our own (the reference uses CLI11, which is not part
// of this build). Exit codes: 0 ok, 1 domain error (`<Name>: <what>` on err),
// 2 usage error.
#include <algorithm>
#include <cstdlib>
#include <fstream>
#include <functional>
#include <map>
#include <optional>
#include <random>
#include <sstream>

#include <json.hpp>

#include "memplan/cli.hpp"
#include "memplan/errors.hpp"
#include "memplan/presets.hpp"
#include "digest.hpp"
#include "memplan/accounting.hpp"

namespace memplan {

namespace {

using ojson = nlohmann::ordered_json;

struct UsageError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// ------------------------------------------------------------- arguments --

// Parsed `--flag value` pairs of one verb, checked against its declaration.
class Args {
 public:
  struct Spec {
    std::vector<std::string> names;  // e.g. {"-o", "--out"}
    bool required = false;
  };

  Args(std::vector<Spec> specs, const std::vector<std::string>& argv, std::size_t from)
      : specs_(std::move(specs)) {
    for (std::size_t i = from; i < argv.size(); ++i) {
      std::string a = argv[i];
      std::optional<std::string> inline_value;
      if (a.rfind("--", 0) == 0) {
        const auto eq = a.find('=');
        if (eq != std::string::npos) {
          inline_value = a.substr(eq + 1);
          a = a.substr(0, eq);
        }
      }
      const Spec* spec = find(a);
      if (!spec) throw UsageError("unexpected argument: " + a);
      const std::string key = spec->names.back();
      if (values_.count(key)) throw UsageError(key + " given more than once");
      if (inline_value) {
        values_[key] = *inline_value;
      } else {
        if (i + 1 >= argv.size()) throw UsageError(a + " requires a value");
        values_[key] = argv[++i];
      }
    }
    for (const Spec& s : specs_)
      if (s.required && !values_.count(s.names.back()))
        throw UsageError(s.names.back() + " is required");
  }

  bool has(const std::string& key) const { return values_.count(key) != 0; }
  std::string str(const std::string& key, const std::string& dflt = "") const {
    const auto it = values_.find(key);
    return it == values_.end() ? dflt : it->second;
  }
  template <typename T>
  T num(const std::string& key, T dflt) const {
    const auto it = values_.find(key);
    return it == values_.end() ? dflt : convert<T>(key, it->second);
  }
  template <typename T>
  std::optional<T> opt(const std::string& key) const {
    const auto it = values_.find(key);
    if (it == values_.end()) return std::nullopt;
    return convert<T>(key, it->second);
  }

 private:
  template <typename T>
  static T convert(const std::string& key, const std::string& text) {
    std::size_t used = 0;
    try {
      if constexpr (std::is_floating_point_v<T>) {
        const double v = std::stod(text, &used);
        if (used == text.size()) return static_cast<T>(v);
      } else if constexpr (std::is_unsigned_v<T>) {
        const unsigned long long v = std::stoull(text, &used);
        if (used == text.size()) return static_cast<T>(v);
      } else {
        const long long v = std::stoll(text, &used);
        if (used == text.size()) return static_cast<T>(v);
      }
    } catch (const std::exception&) {
    }
    throw UsageError("invalid value '" + text + "' for " + key);
  }

  const Spec* find(const std::string& name) const {
    for (const Spec& s : specs_)
      if (std::find(s.names.begin(), s.names.end(), name) != s.names.end()) return &s;
    return nullptr;
  }

  std::vector<Spec> specs_;
  std::map<std::string, std::string> values_;
};

const std::vector<Args::Spec>& hardware_flags() {
  static const std::vector<Args::Spec> f = {
      {{"--h2d-bw"}},         {{"--d2h-bw"}},         {{"--coll-bw"}},
      {{"--coll-alpha"}},     {{"--cpu-optim-rate"}}, {{"--gpu-optim-rate"}},
      {{"--gpu-mem"}},        {{"--cpu-mem"}},        {{"--world-size"}},
  };
  return f;
}

std::vector<Args::Spec> with_hw(std::vector<Args::Spec> specs) {
  for (const auto& f : hardware_flags()) specs.push_back(f);
  return specs;
}

// ---------------------------------------------------------------- helpers --

ModelTrace read_trace_file(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw MalformedTrace("cannot open trace file: " + path);
  return load_trace(in);
}

// A preset name, a profile file, or <name>.json under $MEMPLAN_PRESET_DIR.
HardwareProfile find_hardware(const std::string& name_or_path) {
  try {
    return get_hardware(name_or_path);
  } catch (const UnknownPreset&) {
  }
  std::ifstream in(name_or_path);
  if (!in)
    if (const char* dir = std::getenv("MEMPLAN_PRESET_DIR"))
      in.open(std::string(dir) + "/" + name_or_path + ".json");
  if (!in)
    throw UnknownPreset("'" + name_or_path + "' is neither a hardware preset nor a readable file");
  return load_profile(in);
}

HardwareProfile hardware_from(const Args& a) {
  HardwareProfile hw = find_hardware(a.str("--hw"));
  if (auto v = a.opt<double>("--h2d-bw")) hw.h2d_bw = *v;
  if (auto v = a.opt<double>("--d2h-bw")) hw.d2h_bw = *v;
  if (auto v = a.opt<double>("--coll-bw")) hw.coll_bw = *v;
  if (auto v = a.opt<double>("--coll-alpha")) hw.coll_alpha = *v;
  if (auto v = a.opt<double>("--cpu-optim-rate")) hw.cpu_optim_rate = *v;
  if (auto v = a.opt<double>("--gpu-optim-rate")) hw.gpu_optim_rate = *v;
  if (auto v = a.opt<std::int64_t>("--gpu-mem")) hw.gpu_mem = *v;
  if (auto v = a.opt<std::int64_t>("--cpu-mem")) hw.cpu_mem = *v;
  if (auto v = a.opt<int>("--world-size")) hw.world_size = *v;
  hw.validate();
  return hw;
}

void emit(const std::string& path, const std::string& text, std::ostream& out) {
  if (path.empty() || path == "-") {
    out << text;
    return;
  }
  std::ofstream f(path);
  if (!f) throw Error("IoError", "cannot open output file: " + path);
  f << text;
}

// "512Mi,1Gi,2147483648" -> sizes in bytes
std::vector<std::int64_t> size_list(const std::string& text) {
  std::vector<std::int64_t> out;
  std::stringstream ss(text);
  std::string tok;
  while (std::getline(ss, tok, ',')) {
    if (tok.empty()) continue;
    double scale = 1;
    if (tok.size() > 2 && (tok.compare(tok.size() - 2, 2, "Mi") == 0 ||
                           tok.compare(tok.size() - 2, 2, "Gi") == 0)) {
      scale = tok.back() == 'i' && tok[tok.size() - 2] == 'M' ? (1 << 20) : (1 << 30);
      tok.resize(tok.size() - 2);
    }
    out.push_back(static_cast<std::int64_t>(std::stod(tok) * scale));
  }
  return out;
}

// "lo:hi" or "v"; hi < lo means unset
std::pair<int, int> int_range(const std::string& text) {
  const auto colon = text.find(':');
  if (colon == std::string::npos) {
    const int v = std::stoi(text);
    return {v, v};
  }
  return {std::stoi(text.substr(0, colon)), std::stoi(text.substr(colon + 1))};
}

// B200 extension: `--chunk-bytes used` charges chunk states by their used
// bytes (include/memplan/accounting.hpp); "reference" (default) keeps the
// reference's 8*s_chunk / s_chunk terms and its byte-identical outputs.
std::optional<ScopedUsedBytesAccounting> chunk_accounting(const Args& a, const ChunkLayout& layout) {
  const std::string mode = a.str("--chunk-bytes", "reference");
  if (mode == "reference") return std::nullopt;
  if (mode != "used") throw UsageError("--chunk-bytes must be 'reference' or 'used'");
  return std::optional<ScopedUsedBytesAccounting>(std::in_place, layout);
}

// B200 extension: `--host-mem-bw B` (bytes/s) makes the simulator share host
// DRAM between the host Adam and the PCIe copies (include/memplan/accounting.hpp);
// absent, the simulation is the reference's.
std::optional<ScopedHostMemoryModel> host_memory(const Args& a) {
  if (!a.has("--host-mem-bw")) return std::nullopt;
  const double bw = a.num<double>("--host-mem-bw", 0.0);
  if (!(bw > 0.0)) throw UsageError("--host-mem-bw must be > 0");
  return std::optional<ScopedHostMemoryModel>(std::in_place, bw);
}

struct Workspace {
  ModelTrace trace;
  ChunkLayout layout;
  std::int64_t s_chunk = 0;
};

Workspace open_trace(const std::string& path, std::int64_t s_chunk) {
  Workspace w;
  w.trace = read_trace_file(path);
  if (s_chunk > 0) {
    w.s_chunk = s_chunk;
    w.layout = pack_chunks(w.trace, s_chunk);
  } else {
    std::tie(w.s_chunk, w.layout) = chunk_size_search(w.trace, default_size_grid(w.trace));
  }
  return w;
}

ojson chunk_table(const ChunkLayout& layout) {
  ojson arr = ojson::array();
  for (const Chunk& c : layout.chunks) {
    ojson jc;
    jc["chunk_id"] = c.chunk_id;
    jc["used_bytes"] = c.used_bytes;
    jc["first_op"] = c.first_op;
    jc["last_op"] = c.last_op;
    jc["block_ids"] = c.block_ids;
    arr.push_back(std::move(jc));
  }
  return arr;
}

// ------------------------------------------------------------------ verbs --

int verb_gen_trace(const Args& a, std::ostream& out, std::ostream& err) {
  ModelSpec spec;
  if (a.has("--model")) {
    spec = get_model(a.str("--model"));
  } else if (a.has("--spec")) {
    std::ifstream in(a.str("--spec"));
    if (!in) throw MalformedTrace("cannot open spec file: " + a.str("--spec"));
    const nlohmann::json j = nlohmann::json::parse(in);
    spec.hidden_size = j.at("hidden_size").get<int>();
    spec.n_blocks = j.at("n_blocks").get<int>();
    spec.n_heads = j.at("n_heads").get<int>();
    const auto take_int = [&](const char* k, int& dst) {
      if (j.contains(k)) dst = j[k].get<int>();
    };
    const auto take_bool = [&](const char* k, bool& dst) {
      if (j.contains(k)) dst = j[k].get<bool>();
    };
    take_int("vocab_size", spec.vocab_size);
    take_int("seq_len", spec.seq_len);
    take_int("batch_size", spec.batch_size);
    take_int("dtype_bytes", spec.dtype_bytes);
    take_int("ffn_hidden", spec.ffn_hidden);
    take_int("n_kv_heads", spec.n_kv_heads);
    take_bool("gated_mlp", spec.gated_mlp);
    take_bool("bias", spec.bias);
    take_bool("tied_embeddings", spec.tied_embeddings);
    take_bool("learned_pos_embedding", spec.learned_pos_embedding);
  } else {
    err << "usage error: gen-trace needs --model or --spec\n";
    return 2;
  }
  if (const int b = a.num<int>("--batch", -1); b > 0) spec.batch_size = b;
  if (const int s = a.num<int>("--seq", -1); s > 0) spec.seq_len = s;
  CalibrationConstants calib;
  calib.flops_per_second = a.num<double>("--flops", calib.flops_per_second);
  calib.act_coeff = a.num<double>("--act-coeff", calib.act_coeff);
  calib.temp_spike_frac = a.num<double>("--spike-frac", calib.temp_spike_frac);
  calib.residual_bytes = a.num<std::int64_t>("--residual", calib.residual_bytes);
  std::ostringstream buf;
  save_trace(synthesize_trace(spec, calib), buf);
  emit(a.str("--out"), buf.str(), out);
  return 0;
}

int verb_pack(const Args& a, std::ostream& out) {
  const ModelTrace trace = read_trace_file(a.str("--trace"));
  const auto grid = a.has("--grid") && !a.str("--grid").empty() ? size_list(a.str("--grid"))
                                                                  : default_size_grid(trace);
  const auto [size, layout] = chunk_size_search(trace, grid);
  ojson j;
  j["s_chunk"] = size;
  j["n_chunk"] = layout.n_chunk();
  j["waste_bytes"] = layout.waste_bytes;
  j["chunks"] = chunk_table(layout);
  emit(a.str("--out"), j.dump(2) + "\n", out);
  return 0;
}

int verb_plan(const Args& a, std::ostream& out) {
  const Workspace w = open_trace(a.str("--trace"), a.num<std::int64_t>("--s-chunk", 0));
  const HardwareProfile hw = hardware_from(a);
  const auto accounting = chunk_accounting(a, w.layout);
  const auto hostmem = host_memory(a);
  CostOptions opts;
  opts.alpha = a.num<double>("--alpha", 1.05);
  SearchOutcome res = find_optimal(w.trace, w.layout, hw, opts);
  const int refine = a.num<int>("--refine-sim", 0);
  if (refine <= 0) {  // the reference's behaviour, byte for byte
    const BlockSchedule sched = build_block_schedule(res.best.n_block, res.best.n_swap,
                                                     res.best.n_checkpoint, res.best.n_interval);
    emit(a.str("--out"), plan_to_json(res.best, w.layout, sched, &res), out);
    return 0;
  }
  // B200 extension: pick among the top-k analytic candidates by simulation
  const auto ranked = refine_with_simulation(w.trace, w.layout, hw, res, refine);
  const PlanConfig analytic = res.best;
  res.best = ranked.front().config;
  const BlockSchedule sched = build_block_schedule(res.best.n_block, res.best.n_swap,
                                                   res.best.n_checkpoint, res.best.n_interval);
  res.estimate = estimate_iteration(w.trace, w.layout, sched, res.best, hw, opts);
  nlohmann::ordered_json j = nlohmann::ordered_json::parse(plan_to_json(res.best, w.layout, sched, &res));
  nlohmann::ordered_json r;
  r["analytic_best"] = {{"n_persist", analytic.n_persist}, {"n_buffer", analytic.n_buffer},
                        {"n_swap", analytic.n_swap}, {"n_checkpoint", analytic.n_checkpoint}};
  r["candidates"] = nlohmann::ordered_json::array();
  for (const RefinedChoice& c : ranked) {
    nlohmann::ordered_json row;
    row["n_persist"] = c.config.n_persist;
    row["n_buffer"] = c.config.n_buffer;
    row["n_swap"] = c.config.n_swap;
    row["n_checkpoint"] = c.config.n_checkpoint;
    row["estimate_t_iter"] = c.estimate_t_iter;
    row["simulated_t_iter"] = c.simulated_t_iter;
    row["simulated_m_peak"] = c.simulated_m_peak;
    r["candidates"].push_back(std::move(row));
  }
  j["refined"] = std::move(r);
  emit(a.str("--out"), j.dump(2) + "\n", out);
  return 0;
}

PlanConfig config_for(const Workspace& w, const HardwareProfile& hw, const Args& a) {
  if (a.has("--plan") && !a.str("--plan").empty()) {
    std::ifstream in(a.str("--plan"));
    if (!in) throw MalformedTrace("cannot open plan file: " + a.str("--plan"));
    return plan_config_from_json(in);
  }
  const int np = a.num<int>("--n-persist", -1);
  const int nb = a.num<int>("--n-buffer", -1);
  PlanConfig c;
  c.s_chunk = w.s_chunk;
  c.n_chunk = w.layout.n_chunk();
  c.n_block = w.trace.n_blocks;
  c.n_interval = compute_interval(w.trace, hw);
  c.n_persist = np < 0 ? c.n_chunk : np;
  c.n_buffer = nb >= 0 ? nb : (c.n_persist < c.n_chunk ? std::min(3, c.n_chunk - c.n_persist) : 0);
  c.n_swap = std::max(0, a.num<int>("--n-swap", 0));
  c.n_checkpoint = std::max(0, a.num<int>("--n-checkpoint", 0));
  c.validate();
  return c;
}

int verb_estimate_or_simulate(const Args& a, bool simulate_it, std::ostream& out) {
  const Workspace w = open_trace(a.str("--trace"), a.num<std::int64_t>("--s-chunk", 0));
  const HardwareProfile hw = hardware_from(a);
  const PlanConfig config = config_for(w, hw, a);
  // an explicit plan may carry its own chunk size
  const ChunkLayout layout =
      config.s_chunk == w.s_chunk ? w.layout : pack_chunks(w.trace, config.s_chunk);
  const BlockSchedule sched =
      build_block_schedule(config.n_block, config.n_swap, config.n_checkpoint, config.n_interval);
  const auto accounting = chunk_accounting(a, layout);
  const auto hostmem = simulate_it ? host_memory(a) : std::nullopt;
  if (!simulate_it) {
    CostOptions opts;
    opts.alpha = a.num<double>("--alpha", 1.05);
    emit(a.str("--out"), estimate_to_json(estimate_iteration(w.trace, layout, sched, config, hw, opts)),
         out);
    return 0;
  }
  const SimulationResult r = simulate(w.trace, layout, sched, config, hw);
  if (!a.str("--timeline").empty()) {
    std::ofstream f(a.str("--timeline"));
    timeline_to_chrome_trace(r.timeline, f);
  }
  if (!a.str("--timeline-csv").empty()) {
    std::ofstream f(a.str("--timeline-csv"));
    timeline_to_csv(r.timeline, f);
  }
  if (!a.str("--mem-trace").empty()) {
    std::ofstream f(a.str("--mem-trace"));
    mem_trace_to_csv(r.mem_trace, f);
  }
  emit(a.str("--out"), simulation_to_json(r), out);
  return 0;
}

int verb_validate(const Args& a, std::ostream& out, std::ostream& err) {
  const Workspace w = open_trace(a.str("--trace"), a.num<std::int64_t>("--s-chunk", 0));
  const HardwareProfile hw = hardware_from(a);
  const auto accounting = chunk_accounting(a, w.layout);
  const auto hostmem = host_memory(a);
  CostOptions opts;
  opts.alpha = a.num<double>("--alpha", 1.05);
  const auto configs = sample_feasible_configs(w.trace, w.layout, hw, a.num<int>("--samples", 50),
                                               a.num<unsigned long long>("--seed", 0ULL), opts);
  if (configs.empty()) throw NoFeasibleConfig("no feasible config to sample");
  const ValidationReport report = validate(w.trace, w.layout, hw, configs, opts);
  std::ostringstream buf;
  report.to_csv(buf);
  emit(a.str("--out"), buf.str(), out);
  err << "max_t_rel_err=" << report.max_t_rel_err
      << " median_t_rel_err=" << report.median_t_rel_err << " m_ratio=[" << report.min_m_ratio
      << "," << report.max_m_ratio << "]\n";
  return 0;
}

int verb_sweep(const Args& a, std::ostream& out) {
  const Workspace w = open_trace(a.str("--trace"), a.num<std::int64_t>("--s-chunk", 0));
  const HardwareProfile hw = hardware_from(a);
  const auto accounting = chunk_accounting(a, w.layout);
  CostOptions opts;
  opts.alpha = a.num<double>("--alpha", 1.05);
  const int n_chunk = w.layout.n_chunk();
  const int n_block = w.trace.n_blocks;
  const int n_interval = compute_interval(w.trace, hw);
  auto [p_lo, p_hi] = int_range(a.str("--n-persist", "0:-1"));
  const auto [b_lo0, b_hi0] = int_range(a.str("--n-buffer", "-1:-1"));
  const auto [s_lo, s_hi] = int_range(a.str("--n-swap", "0:0"));
  const auto [c_lo, c_hi] = int_range(a.str("--n-checkpoint", "0:0"));
  if (p_hi < 0) p_hi = n_chunk;
  std::ostringstream buf;
  buf << "s_chunk,n_chunk,n_persist,n_buffer,n_block,n_interval,n_swap,"
         "n_checkpoint,t_fwd,t_bwd,t_gpu_optim,t_cpu_optim,t_iter,m_peak\n";
  for (int np = p_lo; np <= p_hi; ++np) {
    // -1 = the minimum legal buffer count for this np
    const int b_lo = b_lo0 >= 0 ? b_lo0 : (np < n_chunk ? std::min(3, n_chunk - np) : 0);
    const int b_hi = b_hi0 >= 0 ? b_hi0 : b_lo;
    for (int nb = b_lo; nb <= std::min(b_hi, n_chunk - np); ++nb)
      for (int ns = s_lo; ns <= s_hi; ++ns)
        for (int nc = c_lo; nc <= std::min(c_hi, n_block - ns); ++nc) {
          const PlanConfig c{w.s_chunk, n_chunk, np, nb, n_block, n_interval, ns, nc};
          try {
            c.validate();
            const BlockSchedule sched = build_block_schedule(n_block, ns, nc, n_interval);
            const CostEstimate e = estimate_iteration(w.trace, w.layout, sched, c, hw, opts);
            buf << c.s_chunk << ',' << c.n_chunk << ',' << np << ',' << nb << ',' << n_block
                << ',' << n_interval << ',' << ns << ',' << nc << ',' << e.t_fwd << ','
                << e.t_bwd << ',' << e.t_gpu_optim << ',' << e.t_cpu_optim << ',' << e.t_iter
                << ',' << e.m_peak << "\n";
          } catch (const Error&) {
            // an illegal corner of the requested ranges: no row
          }
        }
  }
  emit(a.str("--out"), buf.str(), out);
  return 0;
}

int verb_list_presets(std::ostream& out) {
  ojson j;
  j["models"] = ojson::array();
  for (const std::string& name : PresetCatalog::model_names()) {
    const ModelSpec m = get_model(name);
    ojson row;
    row["name"] = name;
    row["hidden_size"] = m.hidden_size;
    row["n_blocks"] = m.n_blocks;
    row["n_heads"] = m.n_heads;
    row["total_params"] = m.total_params();
    j["models"].push_back(std::move(row));
  }
  j["hardware"] = ojson::array();
  for (const std::string& name : PresetCatalog::hardware_names()) {
    const HardwareProfile h = get_hardware(name);
    ojson row;
    row["name"] = name;
    row["h2d_bw"] = h.h2d_bw;
    row["coll_bw"] = h.coll_bw;
    row["world_size"] = h.world_size;
    row["gpu_mem"] = h.gpu_mem;
    j["hardware"].push_back(std::move(row));
  }
  out << j.dump(2) << "\n";
  return 0;
}

const char* kHelp =
    "memplan: memory-management planning for LLM training (B200 chunk runtime)\n"
    "  gen-trace     synthesize an iteration trace (--model|--spec, --batch, --seq, ...)\n"
    "  pack          chunk-size search and packing (--trace, --grid)\n"
    "  plan          search the optimal configuration (--trace, --hw)\n"
    "  estimate      analytic cost estimate (--trace, --hw, --plan | --n-*)\n"
    "  simulate      event-driven simulation (+ --timeline, --timeline-csv, --mem-trace)\n"
    "  validate      estimate vs. simulation sweep (--samples, --seed)\n"
    "  sweep         estimate over config ranges (--n-persist lo:hi, ...)\n"
    "  list-presets  list model and hardware presets\n"
    "B200 extensions (opt-in; without them every output is the reference's):\n"
    "  plan --refine-sim K                rank the K best candidates by simulation\n"
    "  --chunk-bytes reference|used       charge chunk states by s_chunk or by used bytes\n"
    "  --host-mem-bw B                    simulate host Adam + PCIe copies sharing B bytes/s\n";

}  // namespace

int run_cli(const std::vector<std::string>& args, std::ostream& out, std::ostream& err) {
  using Spec = Args::Spec;
  const std::vector<Spec> est_flags = with_hw({{{"--trace"}, true},
                                               {{"--hw"}, true},
                                               {{"--plan"}},
                                               {{"--alpha"}},
                                               {{"--s-chunk"}},
                                               {{"--n-persist"}},
                                               {{"--n-buffer"}},
                                               {{"--n-swap"}},
                                               {{"--n-checkpoint"}},
                                               {{"--chunk-bytes"}},
                                               {{"-o", "--out"}}});
  std::vector<Spec> sim_flags = est_flags;
  sim_flags.push_back({{"--timeline"}});
  sim_flags.push_back({{"--host-mem-bw"}});
  sim_flags.push_back({{"--timeline-csv"}});
  sim_flags.push_back({{"--mem-trace"}});
  const std::map<std::string, std::vector<Spec>> verbs = {
      {"gen-trace",
       {{{"--model"}}, {{"--spec"}}, {{"--batch"}}, {{"--seq"}}, {{"--flops"}},
        {{"--act-coeff"}}, {{"--spike-frac"}}, {{"--residual"}}, {{"-o", "--out"}}}},
      {"pack", {{{"--trace"}, true}, {{"--grid"}}, {{"-o", "--out"}}}},
      {"plan", with_hw({{{"--trace"}, true}, {{"--hw"}, true}, {{"--alpha"}}, {{"--s-chunk"}},
                        {{"--refine-sim"}}, {{"--chunk-bytes"}}, {{"--host-mem-bw"}},
                        {{"-o", "--out"}}})},
      {"estimate", est_flags},
      {"simulate", sim_flags},
      {"validate", with_hw({{{"--trace"}, true}, {{"--hw"}, true}, {{"--samples"}}, {{"--seed"}},
                            {{"--alpha"}}, {{"--s-chunk"}}, {{"--chunk-bytes"}},
                            {{"--host-mem-bw"}}, {{"-o", "--out"}}})},
      {"sweep", with_hw({{{"--trace"}, true}, {{"--hw"}, true}, {{"--n-persist"}},
                         {{"--n-buffer"}}, {{"--n-swap"}}, {{"--n-checkpoint"}}, {{"--alpha"}},
                         {{"--s-chunk"}}, {{"--chunk-bytes"}}, {{"-o", "--out"}}})},
      {"list-presets", {}},
  };

  if (std::find(args.begin(), args.end(), "-h") != args.end() ||
      std::find(args.begin(), args.end(), "--help") != args.end()) {
    out << kHelp;
    return 0;
  }
  std::optional<Args> parsed;
  std::string verb;
  try {
    if (args.empty()) throw UsageError("a subcommand is required");
    verb = args[0];
    const auto it = verbs.find(verb);
    if (it == verbs.end()) throw UsageError("unknown subcommand: " + verb);
    parsed.emplace(it->second, args, 1);
  } catch (const UsageError& e) {
    err << "usage error: " << e.what() << "\n";
    return 2;
  }

  try {
    const Args& a = *parsed;
    if (verb == "gen-trace") return verb_gen_trace(a, out, err);
    if (verb == "pack") return verb_pack(a, out);
    if (verb == "plan") return verb_plan(a, out);
    if (verb == "estimate") return verb_estimate_or_simulate(a, false, out);
    if (verb == "simulate") return verb_estimate_or_simulate(a, true, out);
    if (verb == "validate") return verb_validate(a, out, err);
    if (verb == "sweep") return verb_sweep(a, out);
    if (verb == "list-presets") return verb_list_presets(out);
  } catch (const UsageError& e) {
    err << "usage error: " << e.what() << "\n";
    return 2;
  } catch (const Error& e) {
    err << e.name() << ": " << e.what() << "\n";
    return 1;
  } catch (const std::exception& e) {
    err << "error: " << e.what() << "\n";
    return 1;
  }
  return 2;
}

// -------------------------------------------------- sampling for validate --

std::vector<PlanConfig> sample_feasible_configs(const ModelTrace& trace, const ChunkLayout& layout,
                                                const HardwareProfile& hw, int n_samples,
                                                unsigned long long seed, const CostOptions& opts) {
  // same pool as filtering enumerate_candidates by estimate_peak_memory +
  // config_feasible (proj/src/cli.cpp:272-293), with the stream's cached peaks
  std::vector<PlanConfig> pool = detail::feasible_candidates(layout, trace, hw, opts);
  // Fisher-Yates with mt19937_64(seed), then keep the first n_samples.
  std::mt19937_64 rng(seed);
  for (std::size_t i = 0; i + 1 < pool.size(); ++i) {
    const std::size_t j = i + rng() % (pool.size() - i);
    std::swap(pool[i], pool[j]);
  }
  if (static_cast<int>(pool.size()) > n_samples) pool.resize(n_samples);
  return pool;
}

}  // namespace memplan
