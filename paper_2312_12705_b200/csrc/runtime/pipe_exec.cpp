#include "runtime/pipe_exec.h"

#include <algorithm>
#include <stdexcept>

#include "trainplan/core.hpp"

namespace gptb200 {

std::vector<PipeAction> pipeline_actions(int pp, int m, int v, int device, int dh_ring, bool forward_only) {
  if (pp < 1 || m < 1 || v < 1 || device < 0 || device >= pp || dh_ring < 1)
    throw std::invalid_argument("pipeline_actions: bad (pp, m, v, device, ring)");
  std::vector<trainplan::PipeOp> ops;
  if (forward_only) {
    for (int mb = 0; mb < m; ++mb)
      for (int c = 0; c < v; ++c) ops.push_back({false, mb, c});
  } else {
    ops = trainplan::pipeline_order(v > 1 ? trainplan::ScheduleKind::Interleaved1F1B : trainplan::ScheduleKind::OneF1B,
                                    pp, m, v, device);
  }
  auto first_vs = [&](int c) { return device == 0 && c == 0; };
  auto last_vs = [&](int c) { return device == pp - 1 && c == v - 1; };
  std::vector<PipeAction> out;
  out.reserve(ops.size());
  std::vector<int> slot_of(static_cast<size_t>(m) * v, -1);
  std::vector<char> busy;
  std::vector<char> head_late(static_cast<size_t>(m) * v, 0);
  int next_dh = 0;
  for (size_t i = 0; i < ops.size(); ++i) {
    const auto& op = ops[i];
    const size_t key = static_cast<size_t>(op.microbatch) * v + op.chunk;
    PipeAction a;
    a.microbatch = op.microbatch;
    a.chunk = op.chunk;
    if (!op.backward) {
      a.kind = PA_FWD;
      int s = 0;
      if (!forward_only) {
        while (s < static_cast<int>(busy.size()) && busy[s]) ++s;
        if (s == static_cast<int>(busy.size())) busy.push_back(0);
        busy[s] = 1;
      }
      slot_of[key] = s;
      a.slot = s;
      if (!first_vs(op.chunk)) a.flags |= PA_RECV;
      if (!last_vs(op.chunk)) a.flags |= PA_SEND;
      if (last_vs(op.chunk)) {
        const bool next_is_bwd = i + 1 < ops.size() && ops[i + 1].backward &&
                                 ops[i + 1].microbatch == op.microbatch && ops[i + 1].chunk == op.chunk;
        if (forward_only || next_is_bwd) a.flags |= PA_HEAD;
        else head_late[key] = 1;
      }
    } else {
      a.kind = PA_BWD;
      a.slot = slot_of[key];
      if (a.slot < 0) throw std::logic_error("pipeline_actions: backward before forward");
      busy[a.slot] = 0;
      a.dh = next_dh;
      next_dh = (next_dh + 1) % dh_ring;
      if (!last_vs(op.chunk)) a.flags |= PA_RECV;
      if (!first_vs(op.chunk)) a.flags |= PA_SEND;
      if (head_late[key]) a.flags |= PA_HEAD_LATE;
      if (op.microbatch == m - 1) a.flags |= PA_LAST_MB;
    }
    out.push_back(a);
  }
  return out;
}

int pipeline_slots(const std::vector<PipeAction>& acts) {
  int n = 1;
  for (const auto& a : acts) n = std::max(n, a.slot + 1);
  return n;
}

}  // namespace gptb200
