// Internal runtime declarations shared by the C-ABI translation units.
#pragma once

#include <algorithm>
#include <string>

#include <cuda_runtime.h>

#include "tcb/kernels.h"

struct tcb_conv_geom;

namespace tcb {

extern thread_local std::string g_last_error;
int fail(int code, const std::string& msg);
int check_cuda(cudaError_t e, const char* what);
ConvGeom to_geom(const tcb_conv_geom& g);
bool geom_valid(const ConvGeom& g, std::string* why);

// Byte layout of a conv plan's workspace: [wgrad split partials | wT | bias column sums].
struct ConvPlanLayout {
    size_t wgrad, wT, colsum, counters;
    size_t off_wT, off_colsum, off_counters, total;
};
ConvPlanLayout conv_plan_layout(const ConvGeom& g, int algo, int prec);
bool algo_applies(const ConvGeom& g, int algo, int prec);

}  // namespace tcb
