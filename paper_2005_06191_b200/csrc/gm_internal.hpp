// Library-internal hooks of gm_capi.cpp for the other host translation units
// (gm_multi.cpp): C++ linkage, not part of the C ABI.
#pragma once

#include "gridmdp_b200.h"

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
