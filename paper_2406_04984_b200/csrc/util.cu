// Small shared host utilities for the sm_100a kernels.
#include <mutex>

#include "common.cuh"

namespace meft_dev {

long long& launch_counter() {
    static thread_local long long n = 0;
    return n;
}

int num_sms() {
    static int n = 0;
    static std::once_flag once;
    std::call_once(once, [] {
        int dev = 0;
        if (cudaGetDevice(&dev) != cudaSuccess ||
            cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0)
            n = 148;
    });
    return n;
}

}  // namespace meft_dev
