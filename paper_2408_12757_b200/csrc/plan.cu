// Automatic parameter search — see planner.cpp for the search.
#include "host.h"

extern "C" nf_status nf_plan_create(const nf_model_cfg* cfg, const nf_batch* shape, const nf_curve_point* pts,
                                    int32_t n_pts, const nf_plan_opts* opts, nf_plan** out) {
  (void)cfg; (void)shape; (void)pts; (void)n_pts; (void)opts; (void)out;
  return nf::set_error(NF_EUNSUPPORTED, "nf_plan_create: autosearch not built yet");
}
