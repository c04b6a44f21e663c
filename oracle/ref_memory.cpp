// Footprint-model oracle driver — TEST INFRASTRUCTURE ONLY. Links the reference library compiled
// from /root/reference/proj/src (oracle/_ref) and prints its answers for the shared case list
// (tests/cpp/memory_cases.inc); `make -C oracle golden` commits them as tests/golden/ref_memory.json.
#include "../tests/cpp/memory_cases.inc"

int main() {
  memory_cases::print_all();
  return 0;
}
