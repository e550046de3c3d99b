// Product build of the planner C-ABI (prefix rp_); see cabi_planner.inc.
#include "cabi_planner.inc"

extern "C" __attribute__((visibility("default"))) const char* rp_version(void) { return "roundpipe-b200 0.1 (sm_100a)"; }
