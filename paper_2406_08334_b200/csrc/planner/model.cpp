// Planner data model: trace invariants and statistics, model-shape synthesis,
// the preset catalog, and the link cost primitives.
//
// Behavioural sources (the reference is the spec; this file is a clean-room
// restatement with the same observable results):
//   trace validation / stats   proj/src/trace.cpp:20-95
//   synthesis (8 ops/block)    proj/src/trace.cpp:194-344
//   presets                    proj/src/presets.cpp:11-133
//   alpha-beta link model      proj/src/hardware.cpp:12-43
#include <algorithm>
#include <cmath>
#include <map>
#include <string>

#include "memplan/errors.hpp"
#include "memplan/hardware.hpp"
#include "memplan/presets.hpp"
#include "memplan/trace.hpp"

namespace memplan {

// ------------------------------------------------------------------ trace --

namespace {

[[noreturn]] void bad_op(const std::string& what, int idx) {
  throw InvariantViolation(what + " (operator index " + std::to_string(idx) + ")");
}

}  // namespace

void ModelTrace::validate() const {
  if (ops.empty()) throw InvariantViolation("trace has no operators");
  if (m_fwd < 0) throw InvariantViolation("m_fwd must be non-negative");
  if (n_blocks < 0) throw InvariantViolation("n_blocks must be non-negative");
  int last_block = -1;
  int idx = 0;
  for (const OperatorRecord& op : ops) {
    if (op.index != idx) bad_op("indices must be contiguous 0..len-1", idx);
    if (op.t_fwd < 0) bad_op("t_fwd must be >= 0", idx);
    if (op.t_bwd < 0) bad_op("t_bwd must be >= 0", idx);
    if (op.param_bytes < 0) bad_op("param_bytes must be >= 0", idx);
    if (op.act_bytes < 0) bad_op("act_bytes must be >= 0", idx);
    if (op.d_peak_op < std::max<std::int64_t>(0, op.d_cur_op))
      bad_op("d_peak_op must be >= max(0, d_cur_op)", idx);
    if (op.d_peak_prior < std::max<std::int64_t>(0, op.d_cur_prior))
      bad_op("d_peak_prior must be >= max(0, d_cur_prior)", idx);
    if (op.block_id.has_value()) {
      const int b = *op.block_id;
      if (b < 0 || b >= n_blocks) bad_op("block_id outside [0, n_blocks)", idx);
      if (b < last_block) bad_op("block_id values must be non-decreasing", idx);
      last_block = b;
    }
    ++idx;
  }
}

int ModelTrace::dtype_bytes() const {
  const auto it = meta.find("dtype_bytes");
  if (it == meta.end()) return 2;
  try {
    const int v = std::stoi(it->second);
    return v > 0 ? v : 2;
  } catch (...) {
    return 2;
  }
}

std::int64_t ModelTrace::total_param_bytes() const {
  std::int64_t sum = 0;
  for (const auto& op : ops) sum += op.param_bytes;
  return sum;
}

std::int64_t ModelTrace::total_act_bytes() const {
  std::int64_t sum = 0;
  for (const auto& op : ops) sum += op.act_bytes;
  return sum;
}

double ModelTrace::total_fwd_time() const {
  double sum = 0;
  for (const auto& op : ops) sum += op.t_fwd;
  return sum;
}

double ModelTrace::total_bwd_time() const {
  double sum = 0;
  for (const auto& op : ops) sum += op.t_bwd;
  return sum;
}

std::int64_t block_activation_bytes(const ModelTrace& trace, int block) {
  if (block < 0 || block >= trace.n_blocks)
    throw BlockOutOfRange("block " + std::to_string(block) + " outside [0, " +
                          std::to_string(trace.n_blocks) + ")");
  std::int64_t sum = 0;
  for (const auto& op : trace.ops)
    if (op.block_id == block) sum += op.act_bytes;
  return sum;
}

// --------------------------------------------------------------- synthesis --

void ModelSpec::validate() const {
  const bool positive = hidden_size > 0 && n_blocks > 0 && n_heads > 0 && vocab_size > 0 &&
                        seq_len > 0 && batch_size > 0 && dtype_bytes > 0;
  if (!positive) throw InvariantViolation("all ModelSpec fields must be positive");
  if (hidden_size % n_heads != 0)
    throw InvariantViolation("hidden_size must be divisible by n_heads");
  if (n_kv_heads != 0 && n_heads % n_kv_heads != 0)
    throw InvariantViolation("n_heads must be divisible by n_kv_heads");
}

namespace {

// One operator of the fixed per-block sequence.
struct BlockOp {
  const char* name;
  std::int64_t params;     // elements
  double flops;            // forward FLOPs
  std::int64_t act_bytes;  // retained activation (before act_coeff)
};

// The transformer block as 8 hooked operators: pre-norm attention (norm,
// fused QKV projection, attention core, output projection) and pre-norm MLP
// (norm, up[+gate], activation, down). Shapes follow GPT-2 / Llama.
std::vector<BlockOp> transformer_block(const ModelSpec& m) {
  const std::int64_t h = m.hidden_size;
  const std::int64_t ffn = m.ffn_hidden > 0 ? m.ffn_hidden : 4 * h;
  const std::int64_t kv_width = m.n_kv_heads > 0 ? (h / m.n_heads) * m.n_kv_heads : h;
  const std::int64_t qkv_out = h + 2 * kv_width;
  const std::int64_t up_out = m.gated_mlp ? 2 * ffn : ffn;
  const std::int64_t norm_params = m.bias ? 2 * h : h;
  const double tokens = static_cast<double>(m.batch_size) * m.seq_len;
  const double tok_h = static_cast<double>(m.batch_size) * m.seq_len * h;
  const std::int64_t bytes_per_token =
      static_cast<std::int64_t>(m.batch_size) * m.seq_len * m.dtype_bytes;
  const auto bias_of = [&](std::int64_t width) -> std::int64_t { return m.bias ? width : 0; };

  return {
      {"attn_norm", norm_params, 8 * tok_h, bytes_per_token * h},
      {"attn_qkv", h * qkv_out + bias_of(qkv_out), 2 * tok_h * static_cast<double>(qkv_out),
       bytes_per_token * qkv_out},
      {"attn_core", 0, 4 * tokens * static_cast<double>(m.seq_len) * h, bytes_per_token * h},
      {"attn_out", h * h + bias_of(h), 2 * tok_h * static_cast<double>(h), bytes_per_token * h},
      {"mlp_norm", norm_params, 8 * tok_h, bytes_per_token * h},
      {"mlp_up", h * up_out + bias_of(up_out), 2 * tok_h * static_cast<double>(up_out),
       bytes_per_token * up_out},
      {"mlp_act", 0, 4 * tokens * static_cast<double>(ffn), bytes_per_token * ffn},
      {"mlp_down", ffn * h + bias_of(h), 2 * tok_h * static_cast<double>(ffn),
       bytes_per_token * h},
  };
}

std::int64_t embedding_params(const ModelSpec& m) {
  std::int64_t e = static_cast<std::int64_t>(m.vocab_size) * m.hidden_size;
  if (m.learned_pos_embedding) e += static_cast<std::int64_t>(m.seq_len) * m.hidden_size;
  return e;
}

}  // namespace

std::int64_t ModelSpec::params_per_block() const {
  std::int64_t sum = 0;
  for (const BlockOp& op : transformer_block(*this)) sum += op.params;
  return sum;
}

std::int64_t ModelSpec::total_params() const {
  const std::int64_t head =
      tied_embeddings ? 0 : static_cast<std::int64_t>(vocab_size) * hidden_size;
  return embedding_params(*this) + head + static_cast<std::int64_t>(n_blocks) * params_per_block();
}

ModelTrace synthesize_trace(const ModelSpec& spec, const CalibrationConstants& calib) {
  spec.validate();
  if (calib.flops_per_second <= 0)
    throw InvariantViolation("calibration throughput must be positive");
  if (calib.act_coeff <= 0) throw InvariantViolation("activation coefficient must be positive");
  if (calib.temp_spike_frac < 0)
    throw InvariantViolation("temp spike fraction must be non-negative");
  if (calib.residual_bytes < 0) throw InvariantViolation("residual bytes must be non-negative");

  ModelTrace t;
  t.n_blocks = spec.n_blocks;
  t.m_fwd = calib.residual_bytes;
  t.meta = {
      {"generator", "synthesize_trace"},
      {"hidden_size", std::to_string(spec.hidden_size)},
      {"n_heads", std::to_string(spec.n_heads)},
      {"vocab_size", std::to_string(spec.vocab_size)},
      {"seq_len", std::to_string(spec.seq_len)},
      {"batch_size", std::to_string(spec.batch_size)},
      {"dtype_bytes", std::to_string(spec.dtype_bytes)},
      {"flops_per_second", std::to_string(calib.flops_per_second)},
  };

  // Appends one operator; the transient spike is a fraction of `spike_of`
  // (the op's own retained bytes unless an explicit basis is given).
  const auto emit = [&](std::string name, std::optional<int> block, std::int64_t elems,
                        double flops, std::int64_t raw_act, std::int64_t spike_basis) {
    OperatorRecord op;
    op.index = static_cast<int>(t.ops.size());
    op.name = std::move(name);
    op.block_id = block;
    op.param_bytes = elems * spec.dtype_bytes;
    op.t_fwd = flops / calib.flops_per_second;
    op.t_bwd = 2.0 * op.t_fwd;
    op.act_bytes = static_cast<std::int64_t>(std::floor(calib.act_coeff * static_cast<double>(raw_act)));
    const std::int64_t basis = spike_basis != 0 ? spike_basis : op.act_bytes;
    op.d_peak_op = static_cast<std::int64_t>(
        std::floor(calib.temp_spike_frac * static_cast<double>(basis)));
    t.ops.push_back(std::move(op));
  };

  const double tokens = static_cast<double>(spec.batch_size) * spec.seq_len;
  const std::int64_t bytes_per_token =
      static_cast<std::int64_t>(spec.batch_size) * spec.seq_len * spec.dtype_bytes;

  emit("embedding", std::nullopt, embedding_params(spec), 2 * tokens * spec.hidden_size,
       bytes_per_token * spec.hidden_size, 0);
  const std::vector<BlockOp> block = transformer_block(spec);
  for (int b = 0; b < spec.n_blocks; ++b)
    for (const BlockOp& op : block)
      emit(std::string(op.name) + "." + std::to_string(b), b, op.params, op.flops, op.act_bytes, 0);

  const std::int64_t logits = static_cast<std::int64_t>(spec.batch_size) * spec.seq_len *
                              spec.vocab_size * spec.dtype_bytes;
  const std::int64_t head_params =
      spec.tied_embeddings ? 0 : static_cast<std::int64_t>(spec.vocab_size) * spec.hidden_size;
  emit("lm_head", std::nullopt, head_params,
       2 * tokens * static_cast<double>(spec.hidden_size) * spec.vocab_size, logits, 0);
  emit("cross_entropy", std::nullopt, 0, 5 * tokens * static_cast<double>(spec.vocab_size), 0,
       logits);

  t.validate();
  return t;
}

// ---------------------------------------------------------------- presets --

namespace {

ModelSpec gpt2_shape(int hidden, int blocks, int heads) {
  ModelSpec s;
  s.hidden_size = hidden;
  s.n_blocks = blocks;
  s.n_heads = heads;
  return s;
}

ModelSpec llama_shape(int hidden, int blocks, int heads, int ffn, int kv_heads) {
  ModelSpec s = gpt2_shape(hidden, blocks, heads);
  s.vocab_size = 32000;
  s.ffn_hidden = ffn;
  s.n_kv_heads = kv_heads;
  s.gated_mlp = true;
  s.bias = false;
  s.tied_embeddings = false;
  s.learned_pos_embedding = false;
  return s;
}

const std::map<std::string, ModelSpec>& models() {
  // OPT uses the GPT-2 block shape (4h MLP with biases, learned positions).
  static const std::map<std::string, ModelSpec> m = {
      {"gpt2-1b", gpt2_shape(1536, 32, 16)},
      {"gpt2-10b", gpt2_shape(4096, 48, 32)},
      {"gpt2-15b", gpt2_shape(8192, 18, 64)},
      {"gpt2-20b", gpt2_shape(8192, 24, 64)},
      {"gpt2-30b", gpt2_shape(8192, 36, 64)},
      {"gpt2-40b", gpt2_shape(8192, 50, 64)},
      {"opt-13b", gpt2_shape(5120, 40, 40)},
      {"opt-30b", gpt2_shape(7168, 48, 56)},
      {"mistral-7b", llama_shape(4096, 32, 32, 14336, 8)},
      {"llama-13b", llama_shape(5120, 40, 40, 13824, 40)},
      {"llama-34b", llama_shape(8192, 48, 64, 22016, 8)},
  };
  return m;
}

HardwareProfile testbed(double pcie_bw, double coll_bw, int world, std::int64_t gpu_mem,
                        std::int64_t cpu_mem) {
  HardwareProfile hw;
  hw.h2d_bw = pcie_bw;
  hw.d2h_bw = pcie_bw;
  hw.coll_alpha = 20e-6;
  hw.coll_bw = coll_bw;
  hw.world_size = world;
  hw.gpu_mem = gpu_mem;
  hw.cpu_mem = cpu_mem;
  hw.cpu_optim_rate = 0.5e9;  // flagged for calibration (README "Calibration")
  hw.gpu_optim_rate = 1e10;
  return hw;
}

const std::map<std::string, HardwareProfile>& testbeds() {
  // The paper's two testbeds: 4x RTX 3090 over PCIe 3 without NVLink (NCCL
  // ring ~4 GB/s) and 4x A100 80GB over NVLink 3 (300 GB/s).
  static const std::map<std::string, HardwareProfile> m = {
      {"rtx3090x4", testbed(15.8e9, 4e9, 4, 24'000'000'000, 384'000'000'000)},
      {"rtx3090x1", testbed(15.8e9, 4e9, 1, 24'000'000'000, 384'000'000'000)},
      {"a100x4", testbed(31.5e9, 300e9, 4, 80'000'000'000, 1'000'000'000'000)},
      {"a100x1", testbed(31.5e9, 300e9, 1, 80'000'000'000, 1'000'000'000'000)},
  };
  return m;
}

template <typename Map>
std::vector<std::string> keys_of(const Map& m) {
  std::vector<std::string> out;
  out.reserve(m.size());
  for (const auto& kv : m) out.push_back(kv.first);
  return out;
}

}  // namespace

ModelSpec PresetCatalog::model(const std::string& name) {
  const auto& m = models();
  const auto it = m.find(name);
  if (it == m.end()) throw UnknownPreset("no model preset named '" + name + "'");
  return it->second;
}

HardwareProfile PresetCatalog::hardware(const std::string& name) {
  const auto& m = testbeds();
  const auto it = m.find(name);
  if (it == m.end()) throw UnknownPreset("no hardware preset named '" + name + "'");
  return it->second;
}

std::vector<std::string> PresetCatalog::model_names() { return keys_of(models()); }
std::vector<std::string> PresetCatalog::hardware_names() { return keys_of(testbeds()); }
ModelSpec get_model(const std::string& name) { return PresetCatalog::model(name); }
HardwareProfile get_hardware(const std::string& name) { return PresetCatalog::hardware(name); }

// --------------------------------------------------------------- hardware --

void HardwareProfile::validate() const {
  const auto need = [](bool ok, const char* msg) {
    if (!ok) throw InvariantViolation(msg);
  };
  need(h2d_bw > 0, "h2d_bw must be positive");
  need(d2h_bw > 0, "d2h_bw must be positive");
  need(coll_bw > 0, "coll_bw must be positive");
  need(coll_alpha >= 0, "coll_alpha must be non-negative");
  need(world_size >= 1, "world_size must be >= 1");
  need(gpu_mem > 0, "gpu_mem must be positive");
  need(cpu_mem > 0, "cpu_mem must be positive");
  need(cpu_optim_rate > 0, "cpu_optim_rate must be positive");
  need(gpu_optim_rate > 0, "gpu_optim_rate must be positive");
}

double transfer_time(std::int64_t bytes, double bw) {
  if (bw <= 0) throw ZeroBandwidth("transfer bandwidth must be positive");
  return static_cast<double>(bytes) / bw;
}

double gather_time(std::int64_t chunk_bytes, const HardwareProfile& hw) {
  if (hw.world_size <= 1) return 0.0;
  const double w = static_cast<double>(hw.world_size);
  // alpha + bytes * (w-1) / (w * beta), evaluated left to right
  return hw.coll_alpha + static_cast<double>(chunk_bytes) * (w - 1.0) / (w * hw.coll_bw);
}

double reduce_time(std::int64_t chunk_bytes, const HardwareProfile& hw) {
  return gather_time(chunk_bytes, hw);
}

double contended_bandwidth(double base_bw, int n_streams) {
  if (n_streams < 1) throw InvariantViolation("n_streams must be >= 1");
  return base_bw / static_cast<double>(n_streams);
}

}  // namespace memplan
