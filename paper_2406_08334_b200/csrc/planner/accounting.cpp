// Chunk-state accounting (include/memplan/accounting.hpp). The reference
// formulas are proj/src/cost.cpp:10 (8 * s_chunk per persistent chunk),
// proj/include/memplan/cost.hpp:17-21 (s_chunk per buffer) and
// proj/src/search.cpp:135-145 (8 * s_chunk per offloaded chunk on the host).
#include "memplan/accounting.hpp"

#include <algorithm>
#include <string>

#include "memplan/cost.hpp"
#include "memplan/errors.hpp"

namespace memplan {

namespace {

struct UsedBytes {
  bool active = false;
  std::vector<std::int64_t> state_prefix;  // state_prefix[k] = sum_{c<k} 8*used_c
  std::vector<std::int64_t> max_suffix;    // max_suffix[k] = max_{c>=k} used_c (0 past the end)
};

UsedBytes& table() {
  static UsedBytes t;
  return t;
}

const UsedBytes& checked(const PlanConfig& c) {
  const UsedBytes& t = table();
  if (static_cast<int>(t.max_suffix.size()) != c.n_chunk + 1)
    throw InvariantViolation("used-bytes accounting: config has " + std::to_string(c.n_chunk) +
                             " chunks, the layout " +
                             std::to_string(static_cast<int>(t.max_suffix.size()) - 1));
  return t;
}

}  // namespace

bool used_bytes_accounting() { return table().active; }

std::int64_t device_state_bytes(const PlanConfig& c) {
  if (!table().active)
    return persistent_chunk_bytes(c.s_chunk) * c.n_persist +
           buffer_chunk_bytes(c.s_chunk) * c.n_buffer;
  const UsedBytes& t = checked(c);
  return t.state_prefix[c.n_persist] + t.max_suffix[c.n_persist] * c.n_buffer;
}

std::int64_t host_state_bytes(const PlanConfig& c) {
  if (!table().active) return persistent_chunk_bytes(c.s_chunk) * (c.n_chunk - c.n_persist);
  const UsedBytes& t = checked(c);
  return t.state_prefix[c.n_chunk] - t.state_prefix[c.n_persist];
}

ScopedUsedBytesAccounting::ScopedUsedBytesAccounting(const ChunkLayout& layout) {
  UsedBytes& t = table();
  if (t.active) throw InvariantViolation("used-bytes accounting is already active");
  const std::size_t n = layout.chunks.size();
  t.state_prefix.assign(n + 1, 0);
  t.max_suffix.assign(n + 1, 0);
  for (std::size_t c = 0; c < n; ++c)
    t.state_prefix[c + 1] = t.state_prefix[c] + 8 * layout.chunks[c].used_bytes;
  for (std::size_t c = n; c-- > 0;)
    t.max_suffix[c] = std::max(t.max_suffix[c + 1], layout.chunks[c].used_bytes);
  t.active = true;
}

ScopedUsedBytesAccounting::~ScopedUsedBytesAccounting() {
  UsedBytes& t = table();
  t.active = false;
  t.state_prefix.clear();
  t.max_suffix.clear();
}

}  // namespace memplan

namespace memplan {

namespace {
HostMemoryModel& host_model() {
  static HostMemoryModel m;
  return m;
}
}  // namespace

const HostMemoryModel& host_memory_model() { return host_model(); }

ScopedHostMemoryModel::ScopedHostMemoryModel(double bw, double cpu_bytes_per_param) {
  if (!(bw > 0.0) || !(cpu_bytes_per_param > 0.0))
    throw InvariantViolation("host memory model needs bw > 0 and bytes per param > 0");
  if (host_model().bw > 0.0) throw InvariantViolation("host memory model is already active");
  host_model() = HostMemoryModel{bw, cpu_bytes_per_param};
}

ScopedHostMemoryModel::~ScopedHostMemoryModel() { host_model() = HostMemoryModel{}; }

}  // namespace memplan
