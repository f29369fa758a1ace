// dbag_errors.h — shared error reporting of the C-ABI (implemented in
// dbag_capi.cu; read through dbag_last_error / dbag_last_error_info).
#pragma once

#include <cstdint>
#include <string>

namespace dbag {
int set_error(int code, const std::string& msg, int32_t point_id = -1, int32_t cam_id = -1,
              double depth = 0.0);
// Problem::create validation (problem.cpp:66-96) on host arrays (dbag_io.cpp);
// returns a dbag_status and sets *msg.
int validate_problem_arrays(int m, int n, int64_t l, const int32_t* cam, const int32_t* pt,
                            const double* uv, const double* pose, const double* f,
                            const double* pts, std::string* msg);
}  // namespace dbag
