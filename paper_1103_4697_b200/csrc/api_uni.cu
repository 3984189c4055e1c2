// Univariate entry points (Yun / gcd / square-free part): implemented in the next milestone.
#include "api_common.hpp"

extern "C" {
ctg_status ctg_yun_squarefree(const ctg_upoly*, ctg_sqf_buf*, const ctg_opts*) {
  return ctg::guarded([] { throw ctg::ApiError(CTG_UNSUPPORTED, "yun_squarefree: not built yet"); });
}
ctg_status ctg_gcd_univariate(const ctg_upoly*, const ctg_upoly*, ctg_upoly_buf*, const ctg_opts*) {
  return ctg::guarded([] { throw ctg::ApiError(CTG_UNSUPPORTED, "gcd_univariate: not built yet"); });
}
ctg_status ctg_square_free_part(const ctg_upoly*, ctg_upoly_buf*, const ctg_opts*) {
  return ctg::guarded([] { throw ctg::ApiError(CTG_UNSUPPORTED, "square_free_part: not built yet"); });
}
}
