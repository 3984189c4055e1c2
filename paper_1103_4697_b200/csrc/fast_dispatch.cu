// Dispatch of the fast mod-p resultant over the template groups fast_g0..7.cu.
#include "res_common.cuh"

namespace ctg {
#define CTG_DECL(G)                                                             \
  bool dispatch_fast_group_##G(int n, const ResParams& rp, cudaStream_t st); \
  bool dispatch_fused_group_##G(int n, const ResParams& rp, cudaStream_t st);
CTG_DECL(0) CTG_DECL(1) CTG_DECL(2) CTG_DECL(3) CTG_DECL(4) CTG_DECL(5) CTG_DECL(6) CTG_DECL(7)
#undef CTG_DECL

bool dispatch_fast_group(int group, int n, const ResParams& rp, cudaStream_t st) {
  switch (group) {
    case 0: return dispatch_fast_group_0(n, rp, st);
    case 1: return dispatch_fast_group_1(n, rp, st);
    case 2: return dispatch_fast_group_2(n, rp, st);
    case 3: return dispatch_fast_group_3(n, rp, st);
    case 4: return dispatch_fast_group_4(n, rp, st);
    case 5: return dispatch_fast_group_5(n, rp, st);
    case 6: return dispatch_fast_group_6(n, rp, st);
    case 7: return dispatch_fast_group_7(n, rp, st);
    default: return false;
  }
}

bool dispatch_fused_group(int group, int n, const ResParams& rp, cudaStream_t st) {
  switch (group) {
    case 0: return dispatch_fused_group_0(n, rp, st);
    case 1: return dispatch_fused_group_1(n, rp, st);
    case 2: return dispatch_fused_group_2(n, rp, st);
    case 3: return dispatch_fused_group_3(n, rp, st);
    case 4: return dispatch_fused_group_4(n, rp, st);
    case 5: return dispatch_fused_group_5(n, rp, st);
    case 6: return dispatch_fused_group_6(n, rp, st);
    case 7: return dispatch_fused_group_7(n, rp, st);
    default: return false;
  }
}
}  // namespace ctg
