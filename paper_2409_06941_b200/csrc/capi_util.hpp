// Shared helpers of the C-ABI translation units: thread-local error slot,
// exception -> status mapping, and record conversions.
#pragma once

#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "freeride.h"
#include "host/freeride.hpp"

namespace frcapi {

std::string& last_error();
std::string& last_field();

inline int fail(int code, const std::string& msg, const std::string& field = "") {
  last_error() = msg;
  last_field() = field;
  return code;
}

// Thrown by lookup trampolines to carry a caller's status back out.
struct CallbackStatus : std::runtime_error {
  int code;
  explicit CallbackStatus(int c) : std::runtime_error("callback failed"), code(c) {}
};

template <class F>
int guard(F&& f) noexcept {
  try {
    return f();
  } catch (const freeride::ValidationError& e) {
    return fail(FR_ERR_VALIDATION, e.what(), e.field());
  } catch (const freeride::SchemaError& e) {
    return fail(FR_ERR_SCHEMA, e.what(), e.path());
  } catch (const freeride::IllegalTransition& e) {
    return fail(FR_ERR_ILLEGAL_TRANSITION, e.what());
  } catch (const CallbackStatus& e) {
    return e.code;
  } catch (const std::bad_alloc& e) {
    return fail(FR_ERR_INVARIANT, std::string("out of host memory: ") + e.what());
  } catch (const std::exception& e) {
    return fail(FR_ERR_INVARIANT, e.what());
  } catch (...) {
    return fail(FR_ERR_INVARIANT, "unknown exception");
  }
}

inline void copy_id(char* dst, const std::string& s) {
  std::memset(dst, 0, FR_TASK_ID_MAX);
  std::memcpy(dst, s.data(), std::min<std::size_t>(s.size(), FR_TASK_ID_MAX - 1));
}

inline freeride::Bubble bubble_in(const fr_bubble& c) {
  freeride::Bubble b;
  b.stage = c.stage;
  b.epoch = c.epoch;
  b.start = c.start;
  b.duration = c.duration;
  b.available_memory = c.available_memory;
  b.btype = static_cast<freeride::BubbleType>(c.btype);
  return b;
}

inline fr_bubble bubble_out(const freeride::Bubble& b, std::int64_t prev, std::int64_t next) {
  fr_bubble c{};
  c.stage = b.stage;
  c.epoch = b.epoch;
  c.start = b.start;
  c.duration = b.duration;
  c.available_memory = b.available_memory;
  c.btype = static_cast<int32_t>(b.btype);
  c.prev_op = prev;
  c.next_op = next;
  return c;
}

inline freeride::TaskProfile profile_in(const fr_task_profile* p) {
  freeride::TaskProfile tp;
  tp.task_id = std::string(p->task_id, strnlen(p->task_id, FR_TASK_ID_MAX));
  if (p->has_est_per_step) {
    tp.est_per_step_duration = p->est_per_step_duration;
    tp.max_per_step_duration = p->max_per_step_duration;
  }
  tp.est_memory = p->est_memory;
  tp.profiled_steps = p->profiled_steps;
  return tp;
}

inline void profile_out(const freeride::TaskProfile& p, fr_task_profile* out) {
  std::memset(out, 0, sizeof(*out));
  copy_id(out->task_id, p.task_id);
  out->has_est_per_step = p.est_per_step_duration.has_value();
  out->profiled_steps = p.profiled_steps;
  out->est_per_step_duration = p.est_per_step_duration.value_or(0.0);
  out->max_per_step_duration = p.max_per_step_duration.value_or(0.0);
  out->est_memory = p.est_memory;
}

inline freeride::TaskLookup lookup_of(fr_task_lookup_fn fn, void* ctx) {
  return [fn, ctx](const std::string& id) {
    fr_task_view v{};
    const int rc = fn(ctx, id.c_str(), &v);
    if (rc != FR_OK) throw CallbackStatus(rc);
    freeride::TaskView tv;
    tv.state = static_cast<freeride::SideTaskState>(v.state);
    tv.initializing = v.initializing != 0;
    return tv;
  };
}

inline int actions_out(const std::vector<freeride::ManagerAction>& acts, fr_manager_action* out,
                       int32_t cap, int32_t* n_out) {
  *n_out = static_cast<int32_t>(acts.size());
  if (*n_out > cap) return fail(FR_ERR_CAPACITY, "action buffer too small");
  for (std::size_t i = 0; i < acts.size(); ++i) {
    out[i].kind = static_cast<int32_t>(acts[i].kind);
    copy_id(out[i].task_id, acts[i].task_id);
  }
  return FR_OK;
}

}  // namespace frcapi
