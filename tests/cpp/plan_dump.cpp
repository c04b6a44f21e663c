// The product library's answers for the footprint-model case list (tests/cpp/memory_cases.inc),
// compiled against this repo's headers and libtrainplan_b200.so only.
#include "memory_cases.inc"

int main() {
  memory_cases::print_all();
  return 0;
}
