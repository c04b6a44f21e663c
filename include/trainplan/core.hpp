// Umbrella header: the whole trainplan API this library builds on (reference declarations restated
// in arch / cluster / memory / search / pipesim / perf / metrics .hpp, B200 additions in b200.hpp).
#pragma once

#include "trainplan/arch.hpp"
#include "trainplan/b200.hpp"
#include "trainplan/cluster.hpp"
#include "trainplan/memory.hpp"
#include "trainplan/metrics.hpp"
#include "trainplan/perf.hpp"
#include "trainplan/pipesim.hpp"
#include "trainplan/search.hpp"
