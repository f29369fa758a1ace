// dbag_metrics.h — metric extras (dbag_metrics.cu), called by the C-ABI.
#pragma once

#include <string>

#include "../../include/dbag.h"

namespace dbag {
namespace metrics {
int align_similarity(const dbag_param_view* state, const dbag_param_view* reference,
                     int32_t device, double* out_pose, double* out_points, std::string* err);
}  // namespace metrics
}  // namespace dbag
