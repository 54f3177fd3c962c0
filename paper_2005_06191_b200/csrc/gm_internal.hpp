// Library-internal hooks of gm_capi.cpp for the other host translation units
// (gm_multi.cpp): C++ linkage, not part of the C ABI.
#pragma once

#include "gridmdp_b200.h"
#include "gm_kernels.cuh"

#include <functional>
#include <string>

// A result with its tables sized (uninitialised) and the terminal column set
// (run_backward, synthesis.cpp:177-181); `absorbing` (n_states flags) is copied
// for reach specs.
gm_result* gmi_result_new(const gm_model* m, int mode, const uint8_t* absorbing);
// Writable column-major tables of a result (values n_x x (T+1), policy / worst n_x x T).
void gmi_result_tables(gm_result* r, double** values, uint32_t** policy, uint32_t** worst);
// The C ABI's exception -> gm_status mapping.
gm_code gmi_guarded(gm_status* st, const std::function<void()>& f);
// Rethrows a gm_status code as the matching exception type.
[[noreturn]] void gmi_throw(int code, const std::string& msg);
// gm_step_device whose pass-2 epilogue also stores the step's values into other
// devices' value tables (mir: up to gmk::kMaxMirrors peer columns + state intervals).
gm_code gmi_step_device_mirrored(gm_model* m, gm_matrix* tm, int64_t x0, int64_t x1, const double* d_v_next,
                                  double* d_v_out, uint32_t* d_pol, uint32_t* d_wst, void* stream,
                                  const gmk::GmMirror* mir, gm_status* st);
