// capi_internal.h — helpers shared by the translation units behind the C ABI
// (otprg_capi.cpp: single-GPU path; shard_host.cpp: the A-row-sharded path).
// Internal to libotprg.so.
#pragma once
#include <string>

#include <cuda_runtime.h>

#include "../../include/otprg.h"
#include "ctx.h"
#include "kernels.h"

namespace otprg_capi {

int fail(otprg_ctx* ctx, int code, const std::string& msg);
int cuda_fail(otprg_ctx* ctx, cudaError_t e, const char* what);
// solve_assignment / scale_round_costs validation that needs no cost values
int validate_problem(otprg_ctx* ctx, const otprg_problem* p);
// AssignmentInstance::validate for point instances (costs in [0, 1])
int check_points_range(otprg_ctx* ctx, const otprg_problem* p, const double* dpa_orig,
                       const double* dpb_orig);
// exact threshold table for eps on the device (n_out = 0 when it does not fit)
int points_table(otprg_ctx* ctx, double eps, int* n_out);
int launch_finish(otprg_ctx* ctx);
int check_status(otprg_ctx* ctx, const otprg::Ctl& h, bool need_done);
int export_state(otprg_ctx* ctx, otprg_result* r, otprg::Ctl* hout);
// multi-device contexts (shard_host.cpp): shard point instances over ctx->multi
int multi_prepare(otprg_ctx* ctx, const otprg_problem* p);
int multi_solve(otprg_ctx* ctx, otprg_result* res);

}  // namespace otprg_capi

#define CK(expr, what)                                                \
  do {                                                                \
    cudaError_t _e = (expr);                                          \
    if (_e != cudaSuccess) return otprg_capi::cuda_fail(ctx, _e, what); \
  } while (0)
