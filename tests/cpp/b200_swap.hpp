// b200_swap.hpp -- force-included (g++ -include) into UNMODIFIED reference
// translation units (proj/tests/acceptance.cpp, proj/src/verify.cpp) so that
// every call they make to the streaming operators lands on the B200 drop-in
// (include/flashsvd_b200/flashsvd_b200.hpp) instead of the reference CPU code:
// the reference's own acceptance gate and verify suites, run against this
// repo's kernels.  The reference headers are included
// first, so their declarations keep the original names; the macros only
// rename the call sites that follow.  Test infrastructure.
#pragma once
#include "flashsvd/attention.hpp"
#include "flashsvd/encoder.hpp"
#include "flashsvd/ffn.hpp"
#include "flashsvd_b200/flashsvd_b200.hpp"

#define flash_svd_attention b200::flash_svd_attention
#define lowrank_output_projection b200::lowrank_output_projection
#define ffn_v1 b200::ffn_v1
#define ffn_v2 b200::ffn_v2
#define run_layer b200::run_layer
#define run_model b200::run_model
