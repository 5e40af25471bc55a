// esom_host.h -- host-side helpers shared by the translation units of libesom.so.
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

namespace esom_host {
// printf-style message into the thread-local error string; returns code
int set_err(int code, const char* fmt, ...) __attribute__((format(printf, 2, 3)));
int cuda_check(const char* where, int launches = 1);  // also counts our kernel launches
int num_sms();
int max_smem_optin();
size_t resident_limit();
// esom_train.cu: on-chip (cluster) online tick; -1 = shape needs the global-memory kernel
int launch_online_tick_cluster(bool som, const float* X, int d, const int64_t* sample, int B, float* hi,
                               const float* lo, int g, double sigma, double alpha, cudaStream_t st);
}  // namespace esom_host
