// The opaque C handle behind fr_run_trace (freeride.h): a RunTrace from the
// simulated engine (fr_run_experiment) or recorded on the GPU
// (fr_harness_run_trace).
#pragma once

#include "host/freeride.hpp"

struct fr_run_trace {
  freeride::RunTrace t;
};
