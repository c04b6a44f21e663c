// trainplan pipeline schedules — the reference API of
// /root/reference/proj/include/trainplan/pipesim.hpp:8-59, restated for source compatibility.
// The executed per-device order (trainplan::pipeline_order in b200.hpp, bit-exact against the
// reference's simulate()) drives the real 1F1B / interleaved executor; the discrete-event model
// itself (simulate, analytic_bubble, timeline CSV) is the reference planner's and is defined by
// its library (libtrainplan.a).
#pragma once

#include <string>
#include <vector>

namespace trainplan {

enum class ScheduleKind { GPipe, OneF1B, Interleaved1F1B };

struct StageTiming {
  double t_fwd = 1.0;
  double t_bwd = 2.0;
  double t_comm = 0.0;
};

enum class EventKind { Fwd, Bwd, Send, Recv, Idle };

struct TimelineEvent {
  int device = 0;
  EventKind kind = EventKind::Fwd;
  int microbatch = 0;
  int chunk = 0;
  double start = 0.0;
  double end = 0.0;

  friend bool operator==(const TimelineEvent&, const TimelineEvent&) = default;
};

struct IterationTimeline {
  int num_devices = 0;
  std::vector<TimelineEvent> events;
  double makespan = 0.0;
  double bubble_fraction = 0.0;
  double bubble_ratio = 0.0;
};

// Reference planner (defined by libtrainplan.a):
IterationTimeline simulate(ScheduleKind kind, int p, int m, int v, const StageTiming& timing);
double analytic_bubble(ScheduleKind kind, int p, int m, int v);
std::string render_timeline(const IterationTimeline& timeline);
IterationTimeline parse_timeline(const std::string& csv);

}  // namespace trainplan
