// microbench.cu -- the paper's runtime microbenchmarks on B200 (SURVEY.md §8(f)
// NEXT-3 / NEXT-4), include/jacobi3d_microbench.h.  Not part of the Jacobi hot path:
// they measure the launch, overlap and NVLink costs that overdecomposition pays.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdarg>
#include <cstdio>
#include <string>
#include <thread>
#include <vector>

#include "../../include/jacobi3d.h"
#include "../../include/jacobi3d_microbench.h"

namespace jac {
void set_last_error(int code, const char *msg);  // engine.cu
}

namespace {

int mb_fail(int code, const char *fmt, ...)
{
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    jac::set_last_error(code, buf);
    return code;
}

#define MCK(call)                                                                                      \
    do {                                                                                               \
        cudaError_t e_ = (call);                                                                       \
        if (e_ != cudaSuccess) return mb_fail(JAC_ECUDA, "%s: %s", #call, cudaGetErrorString(e_));     \
    } while (0)

double now_us()
{
    return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

__global__ void empty_kernel() {}

__device__ __forceinline__ uint64_t gtimer()
{
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// `work` dependent FMAs per thread; the CTA's first thread stamps start / end.
__global__ void work_kernel(int work, unsigned long long *t_start, unsigned long long *t_end, float *sink)
{
    const uint64_t t0 = gtimer();
    float x = (float)threadIdx.x * 1e-3f, y = 1.0001f;
    for (int i = 0; i < work; ++i) x = fmaf(x, y, 1e-7f);
    if (x == 12345.678f) sink[0] = x;  // keeps the loop alive
    __syncthreads();
    if (threadIdx.x == 0) {
        atomicMin(t_start, (unsigned long long)t0);
        atomicMax(t_end, (unsigned long long)gtimer());
    }
}

// O(n) consumer of a received message (NEXT-3 with compute)
__global__ void consume_kernel(double *p, int64_t n)
{
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        p[i] = p[i] * 1.0000001 + 1e-12;
}

// Byte conservation of the pipelined transfers ("destination buffer region
// equals source region contents"): the source holds a counter-based pattern, every
// delivered 8-byte word is compared with it on the destination device.
__device__ __forceinline__ uint64_t pattern_word(uint64_t i)
{
    uint64_t z = i + 0x5EEDF00DCAFEull;
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

__global__ void fill_pattern_kernel(uint64_t *p, int64_t n)
{
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        p[i] = pattern_word((uint64_t)i);
}

// words [base, base + n) of the source pattern, delivered at p
__global__ void verify_pattern_kernel(const uint64_t *p, int64_t n, int64_t base, unsigned long long *bad)
{
    unsigned long long mine = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        mine += p[i] != pattern_word((uint64_t)(base + i)) ? 8 : 0;
    if (mine) atomicAdd(bad, mine);
}

// Zeroes the destination words [dst_off, dst_off + n) per message, runs `copy_once`
// (one untimed transfer without the consumer kernel), verifies every delivered word.
template <class F>
int verify_delivery(int dst, char *b, const std::vector<std::pair<int64_t, int64_t>> &msgs, F copy_once,
                    int64_t *bad_bytes)
{
    MCK(cudaSetDevice(dst));
    for (const auto &m : msgs) MCK(cudaMemset(b + m.first, 0, m.second));
    MCK(cudaDeviceSynchronize());
    int rc = copy_once();
    if (rc) return rc;
    MCK(cudaSetDevice(dst));
    unsigned long long *bad = nullptr;
    MCK(cudaMalloc(&bad, sizeof *bad));
    MCK(cudaMemset(bad, 0, sizeof *bad));
    for (const auto &m : msgs) {
        const int64_t n = m.second / 8;
        verify_pattern_kernel<<<(unsigned)std::max<int64_t>(1, std::min<int64_t>(1184, (n + 255) / 256)), 256>>>(
            reinterpret_cast<const uint64_t *>(b + m.first), n, m.first / 8, bad);
        MCK(cudaGetLastError());
    }
    unsigned long long h = 0;
    MCK(cudaMemcpy(&h, bad, sizeof h, cudaMemcpyDeviceToHost));
    cudaFree(bad);
    *bad_bytes = (int64_t)h;
    return JAC_OK;
}

typedef CUresult (*PFN_waitValue32)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);

struct Msg {
    const double *src;
    double *dst;
    int64_t n;  // doubles
};

// every CTA walks the message table; message m is split over the grid
__global__ void batched_copy_kernel(const Msg *msgs, int nmsg)
{
    for (int m = 0; m < nmsg; ++m) {
        const Msg g = msgs[m];
        const int64_t n2 = g.n / 2;
        const double2 *s = reinterpret_cast<const double2 *>(g.src);
        double2 *d = reinterpret_cast<double2 *>(g.dst);
        for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n2; i += (int64_t)gridDim.x * blockDim.x)
            d[i] = s[i];
    }
}

__global__ void batched_consume_kernel(const Msg *msgs, int nmsg)
{
    for (int m = 0; m < nmsg; ++m) {
        double *p = msgs[m].dst;
        for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < msgs[m].n; i += (int64_t)gridDim.x * blockDim.x)
            p[i] = p[i] * 1.0000001 + 1e-12;
    }
}

}  // namespace

thread_local int64_t g_mb_verified = 0;  // bytes the last pipeline call checked

extern "C" {

int64_t jac_mb_last_verified_bytes(void) { return g_mb_verified; }

int jac_mb_launch_latency(int32_t device, int32_t iters, double *us)
{
    if (!us || iters < 1) return mb_fail(JAC_EINVAL, "iters must be >= 1, us non-NULL");
    MCK(cudaSetDevice(device));
    cudaStream_t s;
    MCK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    for (int i = 0; i < 50; ++i) {
        empty_kernel<<<1, 32, 0, s>>>();
        MCK(cudaStreamSynchronize(s));
    }
    const double t0 = now_us();
    for (int i = 0; i < iters; ++i) {
        empty_kernel<<<1, 32, 0, s>>>();
        MCK(cudaStreamSynchronize(s));
    }
    *us = (now_us() - t0) / iters;
    cudaStreamDestroy(s);
    return JAC_OK;
}

int jac_mb_overlap(int32_t device, int64_t total_threads, int32_t odf, int32_t work, double *host_us, double *device_us)
{
    if (!host_us || !device_us || odf < 1 || total_threads < odf || work < 0)
        return mb_fail(JAC_EINVAL, "need odf >= 1, total_threads >= odf, work >= 0, non-NULL outputs");
    MCK(cudaSetDevice(device));
    static PFN_waitValue32 waitv = nullptr;
    if (!waitv) {
        void *fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        MCK(cudaGetDriverEntryPoint("cuStreamWaitValue32", &fn, cudaEnableDefault, &q));
        if (!fn) return mb_fail(JAC_ECUDA, "cuStreamWaitValue32 unavailable");
        waitv = (PFN_waitValue32)fn;
    }
    volatile uint32_t *hflag = nullptr;
    MCK(cudaHostAlloc((void **)&hflag, sizeof(uint32_t), cudaHostAllocMapped));
    *hflag = 0;
    void *dflag = nullptr;
    MCK(cudaHostGetDevicePointer(&dflag, (void *)hflag, 0));
    unsigned long long *stamps = nullptr;
    float *sink = nullptr;
    MCK(cudaMalloc(&stamps, 2 * sizeof(unsigned long long)));
    MCK(cudaMalloc(&sink, sizeof(float)));
    const unsigned long long init[2] = {~0ull, 0ull};
    MCK(cudaMemcpy(stamps, init, sizeof init, cudaMemcpyHostToDevice));
    std::vector<cudaStream_t> st(odf);
    for (auto &s : st) MCK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    const int64_t per = total_threads / odf;
    const int block = 256;
    const unsigned grid = (unsigned)std::max<int64_t>(1, (per + block - 1) / block);
    for (int k = 0; k < odf; ++k) {  // everything enqueued up front behind the flag
        if (waitv(st[k], (CUdeviceptr)dflag, 1, CU_STREAM_WAIT_VALUE_GEQ) != CUDA_SUCCESS)
            return mb_fail(JAC_ECUDA, "cuStreamWaitValue32 failed");
        work_kernel<<<grid, block, 0, st[k]>>>(work, stamps, stamps + 1, sink);
        MCK(cudaGetLastError());
    }
    std::this_thread::sleep_for(std::chrono::milliseconds(20));  // let the enqueue settle
    const double t0 = now_us();
    std::atomic_thread_fence(std::memory_order_seq_cst);
    *hflag = 1;  // release every stream at once
    for (auto &s : st) MCK(cudaStreamSynchronize(s));
    *host_us = now_us() - t0;
    unsigned long long out[2];
    MCK(cudaMemcpy(out, stamps, sizeof out, cudaMemcpyDeviceToHost));
    *device_us = (double)(out[1] - out[0]) * 1e-3;
    for (auto &s : st) cudaStreamDestroy(s);
    cudaFree(stamps);
    cudaFree(sink);
    cudaFreeHost((void *)hflag);
    return JAC_OK;
}

int jac_mb_launch_rate(int32_t device, int32_t chares, int32_t threads, double seconds, double *kps)
{
    if (!kps || chares < 1 || threads < 1 || threads > 64 || seconds <= 0)
        return mb_fail(JAC_EINVAL, "need chares >= 1, 1 <= threads <= 64, seconds > 0");
    MCK(cudaSetDevice(device));
    int sms = 0;
    MCK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
    std::vector<long> done(threads, 0);
    std::vector<int> err(threads, 0);
    std::vector<std::thread> pes;
    const double t_end = now_us() + seconds * 1e6;
    for (int p = 0; p < threads; ++p)
        pes.emplace_back([&, p] {
            cudaSetDevice(device);
            std::vector<cudaStream_t> st(chares);
            std::vector<cudaEvent_t> ev(chares);
            std::vector<char> pending(chares, 0);
            for (int c = 0; c < chares; ++c) {
                cudaStreamCreateWithFlags(&st[c], cudaStreamNonBlocking);
                cudaEventCreateWithFlags(&ev[c], cudaEventDisableTiming);
            }
            long n = 0;
            while (now_us() < t_end) {  // the PE's scheduler loop
                for (int c = 0; c < chares; ++c) {
                    if (pending[c]) {
                        if (cudaEventQuery(ev[c]) != cudaSuccess) continue;
                        pending[c] = 0;
                        ++n;
                    }
                    empty_kernel<<<sms * 4, 32, 0, st[c]>>>();  // occupies every SM, no work
                    if (cudaEventRecord(ev[c], st[c]) != cudaSuccess) err[p] = 1;
                    pending[c] = 1;
                }
            }
            for (int c = 0; c < chares; ++c) {
                cudaStreamSynchronize(st[c]);
                cudaStreamDestroy(st[c]);
                cudaEventDestroy(ev[c]);
            }
            done[p] = n;
        });
    for (auto &t : pes) t.join();
    for (int p = 0; p < threads; ++p)
        if (err[p]) return mb_fail(JAC_ECUDA, "launch-rate: event record failed");
    long tot = 0;
    for (long v : done) tot += v;
    *kps = (double)tot / seconds;
    return JAC_OK;
}

int jac_mb_pipeline(int32_t src, int32_t dst, int64_t total_bytes, int32_t odf, int32_t with_compute, double *us)
{
    if (!us || odf < 1 || total_bytes < 8 * (int64_t)odf) return mb_fail(JAC_EINVAL, "need odf >= 1, total_bytes >= 8*odf");
    int ndev = 0;
    MCK(cudaGetDeviceCount(&ndev));
    if (src < 0 || dst < 0 || src >= ndev || dst >= ndev) return mb_fail(JAC_EDEVICE, "src/dst device not present");
    double *a = nullptr, *b = nullptr;
    MCK(cudaSetDevice(src));
    MCK(cudaMalloc(&a, total_bytes));
    fill_pattern_kernel<<<1184, 256>>>(reinterpret_cast<uint64_t *>(a), total_bytes / 8);
    MCK(cudaGetLastError());
    MCK(cudaDeviceSynchronize());
    MCK(cudaSetDevice(dst));
    MCK(cudaMalloc(&b, total_bytes));
    if (src != dst) {
        int can = 0;
        MCK(cudaDeviceCanAccessPeer(&can, dst, src));
        if (!can) return mb_fail(JAC_EDEVICE, "no peer access between devices %d and %d", src, dst);
        cudaError_t e = cudaDeviceEnablePeerAccess(src, 0);
        if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) return mb_fail(JAC_ECUDA, "enable peer access");
        cudaGetLastError();
    }
    std::vector<cudaStream_t> st(odf);
    std::vector<cudaEvent_t> ev(odf);
    for (int k = 0; k < odf; ++k) {
        MCK(cudaStreamCreateWithFlags(&st[k], cudaStreamNonBlocking));
        MCK(cudaEventCreate(&ev[k]));
    }
    cudaStream_t s0;
    cudaEvent_t e0;
    MCK(cudaStreamCreateWithFlags(&s0, cudaStreamNonBlocking));
    MCK(cudaEventCreate(&e0));
    const int64_t chunk = (total_bytes / odf) / 8 * 8;
    auto run = [&]() -> int {
        MCK(cudaEventRecord(e0, s0));
        for (int k = 0; k < odf; ++k) {
            MCK(cudaStreamWaitEvent(st[k], e0, 0));
            char *d = reinterpret_cast<char *>(b) + k * chunk;
            const char *sp = reinterpret_cast<const char *>(a) + k * chunk;
            MCK(cudaMemcpyPeerAsync(d, dst, sp, src, chunk, st[k]));
            if (with_compute) {
                const int64_t n = chunk / 8;
                consume_kernel<<<(unsigned)std::min<int64_t>(1184, (n + 255) / 256), 256, 0, st[k]>>>(
                    reinterpret_cast<double *>(d), n);
                MCK(cudaGetLastError());
            }
            MCK(cudaEventRecord(ev[k], st[k]));
        }
        for (int k = 0; k < odf; ++k) MCK(cudaEventSynchronize(ev[k]));
        return JAC_OK;
    };
    int rc;
    for (int w = 0; w < 3; ++w)
        if ((rc = run())) return rc;
    double best = 1e300;
    for (int rep = 0; rep < 5; ++rep) {
        if ((rc = run())) return rc;
        float mx = 0.f;
        for (int k = 0; k < odf; ++k) {
            float ms = 0.f;
            MCK(cudaEventElapsedTime(&ms, e0, ev[k]));
            mx = std::max(mx, ms);
        }
        best = std::min(best, (double)mx * 1e3);
    }
    *us = best;
    {  // every delivered byte of one more (untimed, consumer-free) transfer
        std::vector<std::pair<int64_t, int64_t>> msgs;
        for (int k = 0; k < odf; ++k) msgs.push_back({k * chunk, chunk});
        const int wc = with_compute;
        with_compute = 0;
        int64_t bad = 0;
        if ((rc = verify_delivery(dst, reinterpret_cast<char *>(b), msgs, run, &bad))) return rc;
        with_compute = wc;
        if (bad) return mb_fail(JAC_ECUDA, "pipeline: %lld of %lld delivered bytes differ from the source",
                                (long long)bad, (long long)(chunk * odf));
        g_mb_verified = chunk * odf;
    }
    for (int k = 0; k < odf; ++k) {
        cudaStreamDestroy(st[k]);
        cudaEventDestroy(ev[k]);
    }
    cudaStreamDestroy(s0);
    cudaEventDestroy(e0);
    cudaFree(b);
    cudaSetDevice(src);
    cudaFree(a);
    return JAC_OK;
}

int jac_mb_pipeline_batched(int32_t src, int32_t dst, int64_t total_bytes, int32_t odf, int32_t with_compute,
                            double *us)
{
    if (!us || odf < 1 || total_bytes < 16 * (int64_t)odf)
        return mb_fail(JAC_EINVAL, "need odf >= 1, total_bytes >= 16*odf");
    int ndev = 0;
    MCK(cudaGetDeviceCount(&ndev));
    if (src < 0 || dst < 0 || src >= ndev || dst >= ndev) return mb_fail(JAC_EDEVICE, "src/dst device not present");
    const int64_t chunk = (total_bytes / odf) / 16 * 16;  // bytes per message
    const int64_t pitch = chunk + 4096;                    // messages live in separate buffers
    char *a = nullptr, *b = nullptr;
    MCK(cudaSetDevice(dst));
    MCK(cudaMalloc(&b, pitch * odf));
    MCK(cudaSetDevice(src));
    MCK(cudaMalloc(&a, pitch * odf));
    fill_pattern_kernel<<<1184, 256>>>(reinterpret_cast<uint64_t *>(a), pitch * odf / 8);
    MCK(cudaGetLastError());
    MCK(cudaDeviceSynchronize());
    if (src != dst) {
        int can = 0;
        MCK(cudaDeviceCanAccessPeer(&can, src, dst));
        if (!can) return mb_fail(JAC_EDEVICE, "no peer access between devices %d and %d", src, dst);
        cudaError_t e = cudaDeviceEnablePeerAccess(dst, 0);
        if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) return mb_fail(JAC_ECUDA, "enable peer access");
        cudaGetLastError();
    }
    std::vector<Msg> h(odf);
    for (int k = 0; k < odf; ++k)
        h[k] = {reinterpret_cast<const double *>(a + k * pitch), reinterpret_cast<double *>(b + k * pitch), chunk / 8};
    Msg *dmsg_src = nullptr, *dmsg_dst = nullptr;
    MCK(cudaMalloc(&dmsg_src, sizeof(Msg) * odf));
    MCK(cudaMemcpy(dmsg_src, h.data(), sizeof(Msg) * odf, cudaMemcpyHostToDevice));
    cudaStream_t ss, sd;
    MCK(cudaStreamCreateWithFlags(&ss, cudaStreamNonBlocking));
    MCK(cudaSetDevice(dst));
    MCK(cudaMalloc(&dmsg_dst, sizeof(Msg) * odf));
    MCK(cudaMemcpy(dmsg_dst, h.data(), sizeof(Msg) * odf, cudaMemcpyHostToDevice));
    MCK(cudaStreamCreateWithFlags(&sd, cudaStreamNonBlocking));
    cudaEvent_t done;
    MCK(cudaSetDevice(src));
    MCK(cudaEventCreateWithFlags(&done, cudaEventDisableTiming));
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, src);
    auto run = [&]() -> int {
        MCK(cudaSetDevice(src));
        batched_copy_kernel<<<sms * 4, 256, 0, ss>>>(dmsg_src, odf);
        MCK(cudaGetLastError());
        MCK(cudaEventRecord(done, ss));
        if (with_compute) {
            MCK(cudaSetDevice(dst));
            MCK(cudaStreamWaitEvent(sd, done, 0));
            batched_consume_kernel<<<sms * 4, 256, 0, sd>>>(dmsg_dst, odf);
            MCK(cudaGetLastError());
            MCK(cudaStreamSynchronize(sd));
        }
        MCK(cudaSetDevice(src));
        MCK(cudaStreamSynchronize(ss));
        return JAC_OK;
    };
    int rc;
    for (int w = 0; w < 3; ++w)
        if ((rc = run())) return rc;
    double best = 1e300;
    for (int rep = 0; rep < 5; ++rep) {
        const double t0 = now_us();
        if ((rc = run())) return rc;
        best = std::min(best, now_us() - t0);
    }
    *us = best;
    {  // every delivered byte of one more (untimed, consumer-free) transfer
        std::vector<std::pair<int64_t, int64_t>> msgs;
        for (int k = 0; k < odf; ++k) msgs.push_back({k * pitch, chunk});
        const int wc = with_compute;
        with_compute = 0;
        int64_t bad = 0;
        if ((rc = verify_delivery(dst, b, msgs, run, &bad))) return rc;
        with_compute = wc;
        if (bad) return mb_fail(JAC_ECUDA, "pipeline_batched: %lld of %lld delivered bytes differ from the source",
                                (long long)bad, (long long)(chunk * odf));
        g_mb_verified = chunk * odf;
    }
    cudaEventDestroy(done);
    cudaStreamDestroy(ss);
    cudaFree(dmsg_src);
    cudaFree(a);
    cudaSetDevice(dst);
    cudaStreamDestroy(sd);
    cudaFree(dmsg_dst);
    cudaFree(b);
    return JAC_OK;
}

}  // extern "C"
