// capi_util.cuh -- status/error plumbing shared by the extern "C" entry points.
#pragma once

#include <cstdarg>
#include <cstdio>
#include <cstring>

#include "../../include/sparseb200.h"
#include "common.cuh"

namespace sb {

inline void clear_error(sb_error *err) {
    if (err) {
        err->code = SB_OK;
        err->row = -1;
        err->iteration = -1;
        err->msg[0] = 0;
    }
}

inline sb_status fail(sb_error *err, sb_status code, const char *fmt, ...) {
    if (err) {
        err->code = code;
        va_list ap;
        va_start(ap, fmt);
        vsnprintf(err->msg, sizeof(err->msg), fmt, ap);
        va_end(ap);
    }
    return code;
}

inline sb_status cuda_fail(sb_error *err, cudaError_t e, const char *where) {
    return fail(err, SB_ERR_CUDA, "%s: %s (%s)", where, cudaGetErrorName(e), cudaGetErrorString(e));
}

#define SB_CUDA(call)                                                 \
    do {                                                              \
        cudaError_t e_ = (call);                                      \
        if (e_ != cudaSuccess) return ::sb::cuda_fail(err, e_, #call); \
    } while (0)

#define SB_GUARD_BEGIN \
    ::sb::clear_error(err); \
    try {
#define SB_GUARD_END                                                          \
    }                                                                         \
    catch (const std::exception &ex) {                                        \
        return ::sb::fail(err, SB_ERR_INVALID_ARGUMENT, "%s", ex.what());     \
    }                                                                         \
    catch (...) {                                                             \
        return ::sb::fail(err, SB_ERR_INVALID_ARGUMENT, "unknown C++ exception"); \
    }

inline cudaStream_t as_stream(sb_stream_t s) { return reinterpret_cast<cudaStream_t>(s); }

// reduction workspace layout: [0, 64) tickets, [64, 128) result scalars,
// [128, 256) scratch (row statistics / first-bad-row flags), [256, ...) partials
constexpr size_t kReduceScratch = 128;
constexpr size_t kReduceHeader = 256;
constexpr size_t kReduceBytes = 256 + 3 * 8 * 4096;

}  // namespace sb
