// Executable form of the per-device pipeline order (trainplan::pipeline_order, which follows
// /root/reference/proj/src/pipesim.cpp:31-91): which activation slot and gradient buffer every
// op uses, which ops receive their input from / send their output to the ring neighbours, and
// where the LM head runs. Stage::step() executes exactly this list; tests/test_pipeline_schedule.py
// replays it for all devices under NCCL rendezvous semantics to prove matching and progress.
//
// Communication model (one process per GPU):
//   * receives are issued on the compute stream right before the op that consumes them;
//   * sends are issued on one side stream per direction right after the op that produced them,
//     so a send never blocks compute; each (direction, ring link) has its own 2-rank NCCL
//     communicator, so activations and gradients never share a FIFO;
//   * an op that reuses a slot / gradient buffer first waits for that buffer's last send.
// Forward activations always travel device p -> (p+1) mod pp, gradients p -> (p-1) mod pp; with
// v > 1 chunks, virtual stage vs = chunk*pp + p, so the wrap link pp-1 -> 0 carries chunk c -> c+1.
#pragma once

#include <vector>

namespace gptb200 {

enum PipeActionKind { PA_FWD = 0, PA_BWD = 1 };
enum PipeActionFlags {
  PA_RECV = 1,       // receive the input (activation or output gradient) first
  PA_SEND = 2,       // send the output (activation or input gradient) afterwards
  PA_HEAD = 4,       // FWD on the last virtual stage: run the LM head + loss now (its BWD follows)
  PA_HEAD_LATE = 8,  // BWD on the last virtual stage whose FWD deferred the head
  PA_LAST_MB = 16,   // BWD of the last microbatch of this chunk: its gradients are final
};

struct PipeAction {
  int kind = PA_FWD, microbatch = 0, chunk = 0, slot = 0, dh = 0, flags = 0;
};

// forward_only: evaluation pass (every microbatch through every chunk, no backward).
std::vector<PipeAction> pipeline_actions(int pp, int m, int v, int device, int dh_ring, bool forward_only);

// Number of activation slots (max microbatch-chunks alive at once on the device).
int pipeline_slots(const std::vector<PipeAction>& acts);

constexpr int kDhRing = 2;  // gradient buffers per device (validated by the rendezvous replay)

}  // namespace gptb200
