// Does a high-priority stream's kernel get the slots a long low-priority grid
// frees as its CTAs retire, and which host calls block while that grid runs?
// (setup-overlap diagnosis for solve_with; not a test)
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o probe_prio tools/probe_prio.cu && ./probe_prio
#include <cuda_runtime.h>
#include <chrono>
#include <cstdio>
#include <thread>

__global__ void k_spin(long long cycles) {
    const long long t0 = clock64();
    while (clock64() - t0 < cycles) {
    }
}
__global__ void k_small(int* x) {
    if (threadIdx.x == 0) atomicAdd(x, 1);
}

static double now_ms() {
    using namespace std::chrono;
    return duration<double, std::milli>(steady_clock::now().time_since_epoch()).count();
}

int main() {
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    cudaStream_t slow, fast;
    cudaStreamCreateWithPriority(&slow, cudaStreamNonBlocking, lo);
    cudaStreamCreateWithPriority(&fast, cudaStreamNonBlocking, hi);
    int* x = nullptr;
    cudaMalloc(&x, 4);
    k_small<<<1, 32, 0, fast>>>(x); // load both kernels before the timed part
    k_spin<<<1, 32, 0, slow>>>(10);
    cudaDeviceSynchronize();
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    // 16 resident CTAs of 256 threads per SM, each spinning ~20 ms; 10 generations ≈ 200 ms
    const int grid = sms * 16 * 10;
    const long long cyc = 20LL * 1900 * 1000;
    for (int mode = 0; mode < 4; ++mode) {
        const double t0 = now_ms();
        k_spin<<<grid, 256, 0, slow>>>(cyc);
        std::this_thread::sleep_for(std::chrono::milliseconds(30));
        const double t1 = now_ms();
        const char* what = "";
        if (mode == 0) {
            what = "kernel on the high-priority stream";
            k_small<<<1, 32, 0, fast>>>(x);
            cudaStreamSynchronize(fast);
        } else if (mode == 1) {
            what = "cudaMalloc 256 MB";
            void* p = nullptr;
            cudaMalloc(&p, 256 << 20);
            cudaFree(p);  // (cudaFree is known to synchronise; timed together)
        } else if (mode == 2) {
            what = "cudaMalloc 256 MB (no free)";
            void* p = nullptr;
            cudaMalloc(&p, 256 << 20);
        } else {
            what = "pageable cudaMemcpyAsync D2H + sync (high-priority stream)";
            int h = 0;
            cudaMemcpyAsync(&h, x, 4, cudaMemcpyDeviceToHost, fast);
            cudaStreamSynchronize(fast);
        }
        const double t2 = now_ms();
        cudaStreamSynchronize(slow);
        const double t3 = now_ms();
        std::printf("%-60s waited %7.1f ms; long grid took %7.1f ms\n", what, t2 - t1, t3 - t0);
    }
    return 0;
}
