// C-ABI plumbing: thread-local error state, device probe, the host RoPE table.
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <string>

#include "common.cuh"

namespace {
thread_local std::string g_error;
}

namespace hph {

int set_error(int code, const char* fmt, ...) {
    char buf[1024];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_error = buf;
    return code;
}

int check_cuda(cudaError_t e, const char* what) {
    if (e == cudaSuccess) return HP_OK;
    return set_error(HP_RUNTIME_ERROR, "%s: CUDA error %s (%s)", what, cudaGetErrorName(e),
                     cudaGetErrorString(e));
}

}  // namespace hph

extern "C" const char* hp_last_error(void) { return g_error.c_str(); }



extern "C" int hp_version(void) { return 1; }

extern "C" int hp_device_available(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n > 0 ? 1 : 0;
}

// build_rope_table (reference tensor.cpp:30-59): freq_i = theta^(-2i/d) and
// angle = p * freq_i in double, cos/sin in double, cast to float — the same
// expressions evaluated by the same libm, so the table is bit-identical.
extern "C" int hp_build_rope_table(int64_t max_pos, int32_t d, float theta, float* cos_out,
                                   float* sin_out) {
    if (d <= 0 || d % 2 != 0)
        return hph::set_error(HP_INVALID_ARGUMENT, "build_rope_table: head_dim must be even and positive, got %d", d);
    if (max_pos <= 0) return hph::set_error(HP_INVALID_ARGUMENT, "build_rope_table: max_position must be >= 1");
    if (!(theta > 0.0f)) return hph::set_error(HP_INVALID_ARGUMENT, "build_rope_table: theta_base must be positive");
    const int half = d / 2;
    for (int i = 0; i < half; ++i) {
        const double freq = std::pow(static_cast<double>(theta),
                                     -2.0 * static_cast<double>(i) / static_cast<double>(d));
        for (int64_t p = 0; p < max_pos; ++p) {
            const double angle = static_cast<double>(p) * freq;
            cos_out[p * half + i] = static_cast<float>(std::cos(angle));
            sin_out[p * half + i] = static_cast<float>(std::sin(angle));
        }
    }
    return HP_OK;
}
