// Shared helpers for libmeshloop_b200: thread-local error string, CUDA checks.
#pragma once
#include <cstdarg>
#include <cstdio>
#include <string>

#include "../../include/meshloop_b200.h"

namespace ml {

void set_error(const char *fmt, ...);
const char *get_error();

}  // namespace ml

#define ML_FAIL(code, ...)              \
    do {                                \
        ::ml::set_error(__VA_ARGS__);   \
        return (code);                  \
    } while (0)

#define ML_CUDA(call)                                                              \
    do {                                                                           \
        cudaError_t err_ = (call);                                                 \
        if (err_ != cudaSuccess)                                                   \
            ML_FAIL(ML_ECUDA, "%s failed: %s", #call, cudaGetErrorString(err_));   \
    } while (0)

// Wrap a body that may throw (std::bad_alloc etc.) so nothing crosses the ABI.
#define ML_GUARD_BEGIN try {
#define ML_GUARD_END                                                   \
    }                                                                  \
    catch (const std::bad_alloc &) {                                   \
        ML_FAIL(ML_ENOMEM, "host allocation failed");                  \
    }                                                                  \
    catch (const std::exception &ex_) {                                \
        ML_FAIL(ML_EINVAL, "%s", ex_.what());                          \
    }
