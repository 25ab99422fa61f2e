// C-ABI over the shared chunk-runtime policy and the planner CLI:
//   ptk_pool_*        memplan::ChunkBufferPool (include/memplan/policy.hpp) for a
//                     host runtime that moves the bytes itself -- the training
//                     loop's chunk pool (paper_2406_08334_b200/offload.py) makes
//                     every residency / slot / eviction decision here, the same
//                     code the simulator and the device executor run;
//   ptk_memplan_run   the memplan command line in process (memplan::run_cli,
//                     proj/include/memplan/cli.hpp:20-35): the planner API for
//                     hosts that cannot link C++ (ctypes / cgo / JNI).
#include <cstdlib>
#include <cstring>
#include <sstream>
#include <string>
#include <vector>

#include "memplan/cli.hpp"
#include "memplan/errors.hpp"
#include "memplan/policy.hpp"
#include "ptk.h"
#include "../ptk_common.h"

struct ptk_pool {
  memplan::ChunkBufferPool pool;
  ptk_pool(int n, int np, int nb) : pool(n, np, nb) {}
};

namespace {

int bad_chunk(const ptk_pool* p, int32_t c, const char* what) {
  if (!p) return ptk::fail(PTK_EINVAL, std::string(what) + ": null pool");
  if (c < 1 || c > p->pool.n_chunk())
    return ptk::fail(PTK_EINVAL, std::string(what) + ": chunk id out of range");
  return PTK_OK;
}

template <class F>
int guarded(const char* what, F&& f) {
  try {
    return f();
  } catch (const memplan::Error& e) {
    return ptk::fail(PTK_EINVAL, std::string(what) + ": " + e.name() + ": " + e.what());
  } catch (const std::exception& e) {
    return ptk::fail(PTK_EINVAL, std::string(what) + ": " + e.what());
  }
}

char* dup(const std::string& s) {
  char* p = static_cast<char*>(std::malloc(s.size() + 1));
  if (p) std::memcpy(p, s.c_str(), s.size() + 1);
  return p;
}

}  // namespace

extern "C" {

int ptk_pool_create(int32_t n_chunk, int32_t n_persist, int32_t n_buffer, ptk_pool** out) {
  if (!out) return ptk::fail(PTK_EINVAL, "ptk_pool_create: null out");
  *out = nullptr;
  return guarded("ptk_pool_create", [&] {
    *out = new ptk_pool(n_chunk, n_persist, n_buffer);
    return PTK_OK;
  });
}

void ptk_pool_destroy(ptk_pool* pool) { delete pool; }

int ptk_pool_grant(ptk_pool* pool, int32_t c, int32_t now, const int32_t* pinned, int32_t n_pinned,
                   int32_t demand, int32_t* slot, int32_t* evicted) {
  if (const int rc = bad_chunk(pool, c, "ptk_pool_grant")) return rc;
  if (!slot || !evicted || n_pinned < 0 || (n_pinned > 0 && !pinned))
    return ptk::fail(PTK_EINVAL, "ptk_pool_grant: bad argument");
  return guarded("ptk_pool_grant", [&] {
    const std::vector<int> pin(pinned, pinned + n_pinned);
    const auto g = pool->pool.grant(c, now, pin, demand != 0);
    *slot = g ? g->slot : -1;
    *evicted = g ? g->evicted : 0;
    return PTK_OK;
  });
}

int ptk_pool_arrived(ptk_pool* pool, int32_t c) {
  if (const int rc = bad_chunk(pool, c, "ptk_pool_arrived")) return rc;
  return guarded("ptk_pool_arrived", [&] {
    pool->pool.arrived(c);
    return PTK_OK;
  });
}

int ptk_pool_release(ptk_pool* pool, int32_t c, int32_t* slot) {
  if (const int rc = bad_chunk(pool, c, "ptk_pool_release")) return rc;
  return guarded("ptk_pool_release", [&] {
    pool->pool.drain_started(c);
    const int s = pool->pool.drain_finished(c);
    if (slot) *slot = s;
    return PTK_OK;
  });
}

int32_t ptk_pool_slot_of(const ptk_pool* pool, int32_t c) {
  if (bad_chunk(pool, c, "ptk_pool_slot_of") != PTK_OK) return -1;
  return pool->pool.slot_of(c);
}

int32_t ptk_pool_chunk_in_slot(const ptk_pool* pool, int32_t s) {
  if (!pool || s < 0 || s >= pool->pool.n_slots()) return 0;
  return pool->pool.chunk_in_slot(s);
}

int32_t ptk_pool_residency(const ptk_pool* pool, int32_t c) {
  if (bad_chunk(pool, c, "ptk_pool_residency") != PTK_OK) return -1;
  return static_cast<int32_t>(pool->pool.where(c));
}

int ptk_memplan_run(int32_t argc, const char* const* argv, char** out, char** err) {
  if (argc < 0 || (argc > 0 && !argv) || !out || !err)
    return ptk::fail(PTK_EINVAL, "ptk_memplan_run: bad argument");
  std::vector<std::string> args(argv, argv + argc);
  std::ostringstream o, e;
  int rc = 0;
  try {
    rc = memplan::run_cli(args, o, e);
  } catch (const std::exception& ex) {
    e << "internal error: " << ex.what() << "\n";
    rc = 1;
  }
  *out = dup(o.str());
  *err = dup(e.str());
  return rc;
}

void ptk_free(void* p) { std::free(p); }

}  // extern "C"
