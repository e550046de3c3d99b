// ORACLE / TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// Builds the reference planner (the unmodified header-only library under
// /root/reference/proj/include/roundpipe) behind the same C-ABI glue the
// product uses, with symbol prefix ref_. The include path puts the reference
// headers first (see oracle/Makefile), so every roundpipe:: algorithm here is
// the reference's own; only the POD marshalling is shared with the product.
#define RP_PREFIX ref_
#include "../paper_2604_27085_b200/csrc/planner/cabi_planner.inc"
