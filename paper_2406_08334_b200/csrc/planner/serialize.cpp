// Planner serialisation: trace / profile / plan JSON, estimate and simulation
// summaries, timeline and memory CSVs, Chrome trace, validation CSV.
//
// Schemas and byte layout follow the reference (the JSON is produced with the
// same nlohmann/json 3.11 library, insertion-ordered, dump(2)):
//   trace JSON        proj/src/trace.cpp:102-189   (unknown keys rejected)
//   profile JSON      proj/src/hardware.cpp:45-96
//   plan / estimate   proj/src/cli.cpp:20-57,211-270
//   CSV / Chrome      proj/src/sim.cpp:750-797
#include <istream>
#include <map>
#include <ostream>
#include <set>
#include <string>

#include <json.hpp>

#include "memplan/cli.hpp"
#include "memplan/errors.hpp"
#include "memplan/hardware.hpp"
#include "memplan/sim.hpp"
#include "memplan/trace.hpp"

namespace memplan {

using ojson = nlohmann::ordered_json;
using json = nlohmann::json;

namespace {

const std::set<std::string>& trace_keys() {
  static const std::set<std::string> k = {"meta", "m_fwd", "n_blocks", "ops"};
  return k;
}

const std::set<std::string>& operator_keys() {
  static const std::set<std::string> k = {"index",       "name",         "block_id",
                                          "t_fwd",       "t_bwd",        "param_bytes",
                                          "act_bytes",   "d_cur_prior",  "d_peak_prior",
                                          "d_cur_op",    "d_peak_op"};
  return k;
}

const std::set<std::string>& profile_keys() {
  static const std::set<std::string> k = {"h2d_bw",  "d2h_bw",  "coll_alpha",
                                          "coll_bw", "world_size", "gpu_mem",
                                          "cpu_mem", "cpu_optim_rate", "gpu_optim_rate"};
  return k;
}

void only_known_keys(const json& j, const std::set<std::string>& allowed, const std::string& where) {
  for (const auto& item : j.items())
    if (!allowed.count(item.key()))
      throw MalformedTrace("unknown key '" + item.key() + "' in " + where);
}

json parse_or_throw(std::istream& in, const char* what) {
  try {
    return json::parse(in);
  } catch (const json::exception& e) {
    throw MalformedTrace(std::string(what) + e.what());
  }
}

OperatorRecord operator_from(const json& jo) {
  only_known_keys(jo, operator_keys(), "operator record");
  OperatorRecord op;
  op.index = jo.at("index").get<int>();
  op.name = jo.at("name").get<std::string>();
  if (jo.contains("block_id") && !jo.at("block_id").is_null())
    op.block_id = jo.at("block_id").get<int>();
  op.t_fwd = jo.at("t_fwd").get<double>();
  op.t_bwd = jo.at("t_bwd").get<double>();
  op.param_bytes = jo.at("param_bytes").get<std::int64_t>();
  op.act_bytes = jo.at("act_bytes").get<std::int64_t>();
  op.d_cur_prior = jo.at("d_cur_prior").get<std::int64_t>();
  op.d_peak_prior = jo.at("d_peak_prior").get<std::int64_t>();
  op.d_cur_op = jo.at("d_cur_op").get<std::int64_t>();
  op.d_peak_op = jo.at("d_peak_op").get<std::int64_t>();
  return op;
}

ojson operator_to(const OperatorRecord& op) {
  ojson jo;
  jo["index"] = op.index;
  jo["name"] = op.name;
  jo["block_id"] = op.block_id ? ojson(*op.block_id) : ojson(nullptr);
  jo["t_fwd"] = op.t_fwd;
  jo["t_bwd"] = op.t_bwd;
  jo["param_bytes"] = op.param_bytes;
  jo["act_bytes"] = op.act_bytes;
  jo["d_cur_prior"] = op.d_cur_prior;
  jo["d_peak_prior"] = op.d_peak_prior;
  jo["d_cur_op"] = op.d_cur_op;
  jo["d_peak_op"] = op.d_peak_op;
  return jo;
}

ojson config_to(const PlanConfig& c) {
  ojson j;
  j["s_chunk"] = c.s_chunk;
  j["n_chunk"] = c.n_chunk;
  j["n_persist"] = c.n_persist;
  j["n_buffer"] = c.n_buffer;
  j["n_block"] = c.n_block;
  j["n_interval"] = c.n_interval;
  j["n_swap"] = c.n_swap;
  j["n_checkpoint"] = c.n_checkpoint;
  return j;
}

PlanConfig config_from(const json& j) {
  PlanConfig c;
  c.s_chunk = j.at("s_chunk").get<std::int64_t>();
  c.n_chunk = j.at("n_chunk").get<int>();
  c.n_persist = j.at("n_persist").get<int>();
  c.n_buffer = j.at("n_buffer").get<int>();
  c.n_block = j.at("n_block").get<int>();
  c.n_interval = j.at("n_interval").get<int>();
  c.n_swap = j.at("n_swap").get<int>();
  c.n_checkpoint = j.at("n_checkpoint").get<int>();
  c.validate();
  return c;
}

ojson estimate_to(const CostEstimate& e) {
  ojson j;
  j["t_fwd"] = e.t_fwd;
  j["t_bwd"] = e.t_bwd;
  j["t_gpu_optim"] = e.t_gpu_optim;
  j["t_cpu_optim"] = e.t_cpu_optim;
  j["t_iter"] = e.t_iter;
  j["m_peak"] = e.m_peak;
  j["m_peak_before_alpha"] = e.m_peak_before_alpha;
  return j;
}

}  // namespace

// ----------------------------------------------------------------- trace --

ModelTrace load_trace(std::istream& in) {
  const json j = parse_or_throw(in, "parse failure: ");
  if (!j.is_object()) throw MalformedTrace("top level must be an object");
  only_known_keys(j, trace_keys(), "trace");
  ModelTrace t;
  try {
    t.m_fwd = j.at("m_fwd").get<std::int64_t>();
    t.n_blocks = j.at("n_blocks").get<int>();
    if (j.contains("meta"))
      for (const auto& item : j.at("meta").items())
        t.meta[item.key()] =
            item.value().is_string() ? item.value().get<std::string>() : item.value().dump();
    const json& ops = j.at("ops");
    if (!ops.is_array()) throw MalformedTrace("ops must be an array");
    t.ops.reserve(ops.size());
    for (const json& jo : ops) t.ops.push_back(operator_from(jo));
  } catch (const json::exception& e) {
    throw MalformedTrace(std::string("field error: ") + e.what());
  }
  t.validate();
  return t;
}

void save_trace(const ModelTrace& trace, std::ostream& out) {
  ojson j;
  j["meta"] = ojson::object();
  for (const auto& [k, v] : trace.meta) j["meta"][k] = v;
  j["m_fwd"] = trace.m_fwd;
  j["n_blocks"] = trace.n_blocks;
  ojson ops = ojson::array();
  for (const auto& op : trace.ops) ops.push_back(operator_to(op));
  j["ops"] = std::move(ops);
  out << j.dump(2) << "\n";
}

// --------------------------------------------------------------- profile --

HardwareProfile load_profile(std::istream& in) {
  const json j = parse_or_throw(in, "profile parse failure: ");
  for (const auto& item : j.items())
    if (!profile_keys().count(item.key()))
      throw MalformedTrace("unknown profile key: " + item.key());
  HardwareProfile hw;
  try {
    hw.h2d_bw = j.at("h2d_bw").get<double>();
    hw.d2h_bw = j.at("d2h_bw").get<double>();
    hw.coll_alpha = j.at("coll_alpha").get<double>();
    hw.coll_bw = j.at("coll_bw").get<double>();
    hw.world_size = j.at("world_size").get<int>();
    hw.gpu_mem = j.at("gpu_mem").get<std::int64_t>();
    hw.cpu_mem = j.at("cpu_mem").get<std::int64_t>();
    hw.cpu_optim_rate = j.at("cpu_optim_rate").get<double>();
    hw.gpu_optim_rate = j.at("gpu_optim_rate").get<double>();
  } catch (const json::exception& e) {
    throw MalformedTrace(std::string("profile field error: ") + e.what());
  }
  hw.validate();
  return hw;
}

void save_profile(const HardwareProfile& hw, std::ostream& out) {
  ojson j;
  j["h2d_bw"] = hw.h2d_bw;
  j["d2h_bw"] = hw.d2h_bw;
  j["coll_alpha"] = hw.coll_alpha;
  j["coll_bw"] = hw.coll_bw;
  j["world_size"] = hw.world_size;
  j["gpu_mem"] = hw.gpu_mem;
  j["cpu_mem"] = hw.cpu_mem;
  j["cpu_optim_rate"] = hw.cpu_optim_rate;
  j["gpu_optim_rate"] = hw.gpu_optim_rate;
  out << j.dump(2) << "\n";
}

// ------------------------------------------------------------------ plan --

std::string plan_to_json(const PlanConfig& config, const ChunkLayout& layout,
                         const BlockSchedule& schedule, const SearchOutcome* outcome) {
  ojson j;
  j["config"] = config_to(config);
  ojson chunks = ojson::array();
  for (const Chunk& c : layout.chunks) {
    ojson jc;
    jc["chunk_id"] = c.chunk_id;
    jc["used_bytes"] = c.used_bytes;
    jc["first_op"] = c.first_op;
    jc["last_op"] = c.last_op;
    jc["block_ids"] = c.block_ids;
    chunks.push_back(std::move(jc));
  }
  j["chunks"] = std::move(chunks);
  j["waste_bytes"] = layout.waste_bytes;
  ojson strategies = ojson::array();
  for (BlockStrategy s : schedule.strategies) strategies.push_back(to_string(s));
  j["strategies"] = std::move(strategies);
  if (outcome != nullptr) {
    j["estimate"] = estimate_to(outcome->estimate);
    ojson search;
    search["n_evaluated"] = outcome->n_evaluated;
    search["n_pruned"] = outcome->n_pruned;
    j["search"] = std::move(search);
    ojson frontier = ojson::array();
    for (const auto& [cfg, t_iter] : outcome->frontier) {
      ojson row = config_to(cfg);
      row["t_iter"] = t_iter;
      frontier.push_back(std::move(row));
    }
    j["frontier"] = std::move(frontier);
  }
  return j.dump(2) + "\n";
}

PlanConfig plan_config_from_json(std::istream& in) {
  const json j = parse_or_throw(in, "plan parse failure: ");
  try {
    return config_from(j.contains("config") ? j.at("config") : j);
  } catch (const json::exception& e) {
    throw MalformedTrace(std::string("plan field error: ") + e.what());
  }
}

std::string estimate_to_json(const CostEstimate& est) { return estimate_to(est).dump(2) + "\n"; }

std::string simulation_to_json(const SimulationResult& r) {
  ojson j;
  j["t_iter"] = r.t_iter;
  j["t_fwd"] = r.t_fwd;
  j["t_bwd"] = r.t_bwd;
  j["t_cpu_optim_span"] = r.t_cpu_optim_span;
  j["m_peak"] = r.m_peak;
  j["n_events"] = r.timeline.size();
  return j.dump(2) + "\n";
}

// ------------------------------------------------------------- CSV / trace --

void ValidationReport::to_csv(std::ostream& out) const {
  out << "n_persist,n_buffer,n_swap,n_checkpoint,est_t_iter,sim_t_iter,"
         "t_rel_err,est_m_peak,sim_m_peak,m_ratio,status\n";
  for (const ValidationRow& r : rows) {
    const PlanConfig& c = r.config;
    out << c.n_persist << ',' << c.n_buffer << ',' << c.n_swap << ',' << c.n_checkpoint << ',';
    if (r.failed) {
      out << ",,,,,," << r.error << "\n";
      continue;
    }
    out << r.est_t_iter << ',' << r.sim_t_iter << ',' << r.t_rel_err << ',' << r.est_m_peak << ','
        << r.sim_m_peak << ',' << r.m_ratio << ",ok\n";
  }
}

void timeline_to_csv(const std::vector<TimelineEvent>& timeline, std::ostream& out) {
  out << "time_ns,resource,event,subject\n";
  for (const TimelineEvent& e : timeline)
    out << e.time_ns << ',' << e.resource << ',' << e.event << ",\"" << e.subject << "\"\n";
}

void timeline_to_chrome_trace(const std::vector<TimelineEvent>& timeline, std::ostream& out) {
  // Instant events; a resource becomes a thread row in order of first use.
  ojson events = ojson::array();
  std::map<std::string, int> row_of;
  for (const TimelineEvent& e : timeline) {
    auto it = row_of.find(e.resource);
    if (it == row_of.end())
      it = row_of.emplace(e.resource, static_cast<int>(row_of.size()) + 1).first;
    ojson ev;
    ev["name"] = e.event + " " + e.subject;
    ev["ph"] = "i";
    ev["ts"] = static_cast<double>(e.time_ns) / 1000.0;
    ev["pid"] = 1;
    ev["tid"] = it->second;
    ev["s"] = "t";
    events.push_back(std::move(ev));
  }
  out << events.dump(1) << "\n";
}

void mem_trace_to_csv(const std::vector<MemSample>& samples, std::ostream& out) {
  out << "time_ns,bytes\n";
  for (const MemSample& s : samples) out << s.time_ns << ',' << s.bytes << "\n";
}

}  // namespace memplan
