// common.cuh — status/error plumbing shared by the libcdsp.so translation units.
#pragma once

#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <string>

#include "cdsp.h"

namespace cdsp {

// Thread-local last-error message (cdsp_last_error()).
void set_error(const char* fmt, ...);
const char* last_error();

inline size_t dtype_size(int32_t dt) { return dt == CDSP_BF16 ? 2 : 4; }
inline bool dtype_ok(int32_t dt) { return dt == CDSP_F32 || dt == CDSP_BF16; }

}  // namespace cdsp

#define CDSP_FAIL(code, ...)            \
    do {                                \
        ::cdsp::set_error(__VA_ARGS__); \
        return (code);                  \
    } while (0)

#define CDSP_REQUIRE(cond, code, ...)            \
    do {                                         \
        if (!(cond)) CDSP_FAIL(code, __VA_ARGS__); \
    } while (0)

#define CDSP_CUDA(call)                                                                     \
    do {                                                                                    \
        cudaError_t e_ = (call);                                                            \
        if (e_ != cudaSuccess)                                                              \
            CDSP_FAIL(CDSP_ERR_CUDA, "%s failed: %s (%s:%d)", #call, cudaGetErrorString(e_), \
                      __FILE__, __LINE__);                                                  \
    } while (0)

#define CDSP_CHECK_STATUS(expr)              \
    do {                                     \
        cdsp_status s_ = (expr);             \
        if (s_ != CDSP_OK) return s_;        \
    } while (0)
