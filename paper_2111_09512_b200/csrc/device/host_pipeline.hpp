// Streaming host-buffer pipeline behind ilug_smooth_host_many /
// ilug_dist_smooth_host_many: copy-in, compute and copy-out of consecutive
// independent steps on three streams with three device slots, so step i's
// smoothing overlaps step i+1's H2D and step i-1's D2H (PCIe is full duplex).
// Three slots, not two: with two, step i+1's copy-in into the slot of step
// i-1 waited for step i-1's copy-out, chaining D2H + H2D (2.4 + 5.1 ms at C2)
// across every other step; the third slot lets the copy-in start as soon as
// the link is free (C2: 6.5 -> 5.2 ms per step, bounded by the 2 x 134 MB
// H2D at 52 GB/s).
#pragma once

#include "../kernels/dev.cuh"

namespace ilug {

struct HostPipeline {
    cudaStream_t in = nullptr, run_st = nullptr, out = nullptr;
    static constexpr int kSlots = 3;
    cudaEvent_t loaded[kSlots] = {}, computed[kSlots] = {}, drained[kSlots] = {};
    DBuf<double> b[kSlots], x[kSlots];

    HostPipeline() = default;
    HostPipeline(const HostPipeline&) = delete;
    HostPipeline& operator=(const HostPipeline&) = delete;
    ~HostPipeline() {
        if (!in) return;
        cudaStreamSynchronize(in), cudaStreamSynchronize(run_st), cudaStreamSynchronize(out);
        for (int k = 0; k < kSlots; ++k)
            cudaEventDestroy(loaded[k]), cudaEventDestroy(computed[k]), cudaEventDestroy(drained[k]);
        cudaStreamDestroy(in), cudaStreamDestroy(run_st), cudaStreamDestroy(out);
    }

    /// step(b_dev, x_dev, stream) applies one step in place on x_dev. A step
    /// whose input (b or x) is the previous step's output buffer (the natural
    /// "smooth again in place" pattern) waits for that output's copy-out, so it
    /// reads the updated values; otherwise copies overlap the neighbours' work.
    template <class Step>
    void run(i64 n, long long count, const double* const* bh, double* const* xh, Step&& step) {
        ensure(n);
        const size_t bytes = static_cast<size_t>(n) * sizeof(double);
        for (long long i = 0; i < count; ++i) {
            if (!bh[i] || !xh[i]) fail_invalid("smooth_host_many: null host buffer");
            const int k = static_cast<int>(i % kSlots);
            // slot k is free once step i-3 is copied out (which follows its compute)
            if (i >= kSlots) ILUG_CUDA(cudaStreamWaitEvent(in, drained[k], 0));
            // reading an earlier step's output: wait for its copy-out (read-after-write
            // on the host buffer; the steps in flight are i-1 and i-2)
            for (long long j = i - 1; j >= 0 && j >= i - (kSlots - 1); --j)
                if (bh[i] == xh[j] || xh[i] == xh[j])
                    ILUG_CUDA(cudaStreamWaitEvent(in, drained[static_cast<int>(j % kSlots)], 0));
            ILUG_CUDA(cudaMemcpyAsync(b[k].p, bh[i], bytes, cudaMemcpyHostToDevice, in));
            ILUG_CUDA(cudaMemcpyAsync(x[k].p, xh[i], bytes, cudaMemcpyHostToDevice, in));
            ILUG_CUDA(cudaEventRecord(loaded[k], in));
            ILUG_CUDA(cudaStreamWaitEvent(run_st, loaded[k], 0));
            step(b[k].p, x[k].p, run_st);
            ILUG_CUDA(cudaEventRecord(computed[k], run_st));
            ILUG_CUDA(cudaStreamWaitEvent(out, computed[k], 0));
            ILUG_CUDA(cudaMemcpyAsync(xh[i], x[k].p, bytes, cudaMemcpyDeviceToHost, out));
            ILUG_CUDA(cudaEventRecord(drained[k], out));
        }
        ILUG_CUDA(cudaStreamSynchronize(out));
        ILUG_CUDA(cudaStreamSynchronize(run_st));
        ILUG_CUDA(cudaStreamSynchronize(in));
    }

private:
    void ensure(i64 n) {
        if (!in) {
            ILUG_CUDA(cudaStreamCreateWithFlags(&in, cudaStreamNonBlocking));
            ILUG_CUDA(cudaStreamCreateWithFlags(&run_st, cudaStreamNonBlocking));
            ILUG_CUDA(cudaStreamCreateWithFlags(&out, cudaStreamNonBlocking));
            for (int k = 0; k < kSlots; ++k) {
                ILUG_CUDA(cudaEventCreateWithFlags(&loaded[k], cudaEventDisableTiming));
                ILUG_CUDA(cudaEventCreateWithFlags(&computed[k], cudaEventDisableTiming));
                ILUG_CUDA(cudaEventCreateWithFlags(&drained[k], cudaEventDisableTiming));
            }
        }
        for (int k = 0; k < kSlots; ++k)
            if (b[k].n != n) b[k].alloc(n), x[k].alloc(n);
    }
};

} // namespace ilug
