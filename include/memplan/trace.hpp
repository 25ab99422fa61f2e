// memplan — drop-in planner API of the B200 chunk runtime.
// Profiled-iteration data model (reference contract: proj/include/memplan/trace.hpp:19-100).
//
// A trace is the per-operator record of one training iteration in forward
// execution order. On the B200 runtime the same schema is filled from real
// hooks (the profiler re-feed); synthesize_trace() produces the deterministic
// GPT-2 / Llama shaped traces the planner tests and benchmarks use.
#pragma once

#include <cstdint>
#include <iosfwd>
#include <map>
#include <optional>
#include <string>
#include <vector>

namespace memplan {

struct OperatorRecord {
  int index = 0;                 // position in forward order, 0..len-1
  std::string name;
  std::optional<int> block_id;   // transformer block; empty for embedding / head / loss
  double t_fwd = 0;              // forward seconds
  double t_bwd = 0;              // backward seconds
  std::int64_t param_bytes = 0;  // parameter payload owned by this operator
  std::int64_t act_bytes = 0;    // activation bytes retained for its backward
  // Backward-phase memory deltas: the *_prior pair is the gap before the
  // operator (unhookable work), the *_op pair is the operator body.
  std::int64_t d_cur_prior = 0;
  std::int64_t d_peak_prior = 0;
  std::int64_t d_cur_op = 0;
  std::int64_t d_peak_op = 0;
};

struct ModelTrace {
  std::vector<OperatorRecord> ops;
  std::int64_t m_fwd = 0;  // residual allocation floor at the end of forward
  int n_blocks = 0;
  std::map<std::string, std::string> meta;

  // Throws InvariantViolation naming the first failing operator index.
  void validate() const;
  // meta["dtype_bytes"] if it parses to a positive int, else 2.
  int dtype_bytes() const;

  std::int64_t total_param_bytes() const;
  std::int64_t total_act_bytes() const;
  double total_fwd_time() const;
  double total_bwd_time() const;
};

struct ModelSpec {
  int hidden_size = 0;
  int n_blocks = 0;
  int n_heads = 0;
  int vocab_size = 50257;
  int seq_len = 1024;
  int batch_size = 8;
  int dtype_bytes = 2;

  int ffn_hidden = 0;      // 0 means 4 * hidden_size
  int n_kv_heads = 0;      // 0 means n_heads (no grouped KV)
  bool gated_mlp = false;  // SwiGLU-style: up + gate projections
  bool bias = true;
  bool tied_embeddings = true;
  bool learned_pos_embedding = true;

  void validate() const;
  std::int64_t params_per_block() const;  // elements
  std::int64_t total_params() const;      // elements
};

struct CalibrationConstants {
  double flops_per_second = 42e12;
  double act_coeff = 1.0;
  double temp_spike_frac = 0.25;
  std::int64_t residual_bytes = 256ll << 20;
};

ModelTrace load_trace(std::istream& in);
void save_trace(const ModelTrace& trace, std::ostream& out);

ModelTrace synthesize_trace(const ModelSpec& spec,
                            const CalibrationConstants& calib = {});

std::int64_t block_activation_bytes(const ModelTrace& trace, int block);

}  // namespace memplan
