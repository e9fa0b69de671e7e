// frames.cu -- C ABI of the synthetic frame generator (frames.cuh):
// mbp_frames_generate_device (the product path: frames made in HBM next to
// the decoder) and mbp_frames_generate (the same code on host threads; used
// to pin the algorithm against numpy on machines without a GPU and to fill
// host buffers for end-to-end runs).
#include "../../include/mbp.h"
#include "frames.cuh"

#include <algorithm>
#include <string>
#include <thread>
#include <vector>

namespace mbp {
int set_error(int code, const char* msg);
}

namespace {

int check_args(int32_t n, const uint32_t* prefix, int32_t prefix_len, int64_t first, int64_t batch, double e,
               const void* keys, const void* noisy, mbp::frames::FrameArgs* A)
{
    using mbp::frames::FrameArgs;
    if (n <= 0) return mbp::set_error(MBP_EINVAL, "n must be positive");
    if (batch < 0 || first < 0) return mbp::set_error(MBP_EINVAL, "first and batch must be >= 0");
    if (!(e > 0.0 && e < 0.5)) return mbp::set_error(MBP_EINVAL, "crossover probability must be in (0, 0.5)");
    if (prefix_len < 0 || prefix_len > (int)(sizeof(A->prefix) / 4) || (prefix_len && !prefix))
        return mbp::set_error(MBP_EINVAL, "prefix must hold 0..21 entropy words");
    if (batch && (!keys || !noisy)) return mbp::set_error(MBP_EINVAL, "null pointer argument");
    *A = FrameArgs{};
    for (int i = 0; i < prefix_len; ++i) A->prefix[i] = prefix[i];
    A->plen = prefix_len;
    A->n = n;
    A->nb = (n + 7) / 8;
    A->first = first;
    A->batch = batch;
    A->e = e;
    return MBP_OK;
}

}  // namespace

int mbp_frames_generate_device(int32_t n, const uint32_t* prefix, int32_t prefix_len, int64_t first,
                               int64_t batch, double e, uint8_t* keys, uint8_t* noisy, void* stream)
{
    mbp::frames::FrameArgs A;
    int rc = check_args(n, prefix, prefix_len, first, batch, e, keys, noisy, &A);
    if (rc || batch == 0) return rc;
    cudaStream_t s = (cudaStream_t)stream;
    mbp::frames::Key2* kbuf = nullptr;
    cudaError_t err = cudaMallocAsync((void**)&kbuf, sizeof(mbp::frames::Key2) * 2 * batch, s);
    if (err != cudaSuccess) { cudaGetLastError(); return mbp::set_error(MBP_ENOMEM, "cudaMallocAsync (frame keys) failed"); }
    mbp::frames::frame_keys_kernel<<<(unsigned)((2 * batch + 255) / 256), 256, 0, s>>>(A, kbuf);
    const long long threads = (long long)((n + 31) / 32) * batch;
    mbp::frames::frame_bits_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, s>>>(A, kbuf, keys, noisy);
    err = cudaGetLastError();
    cudaFreeAsync(kbuf, s);
    if (err != cudaSuccess) return mbp::set_error(MBP_ECUDA, (std::string("frame generator: ") + cudaGetErrorString(err)).c_str());
    return MBP_OK;
}

int mbp_frames_generate(int32_t n, const uint32_t* prefix, int32_t prefix_len, int64_t first, int64_t batch,
                        double e, uint8_t* keys, uint8_t* noisy, int32_t threads)
{
    mbp::frames::FrameArgs A;
    int rc = check_args(n, prefix, prefix_len, first, batch, e, keys, noisy, &A);
    if (rc || batch == 0) return rc;
    const int T = (int)std::max<int64_t>(1, std::min<int64_t>(threads > 0 ? threads : 1, batch));
    const long long words = (n + 31) / 32;
    auto work = [&](int t) {
        for (long long f = t; f < batch; f += T) {
            const auto kk = mbp::frames::frame_key(A.prefix, A.plen, (uint64_t)(first + f), 0);
            const auto kf = mbp::frames::frame_key(A.prefix, A.plen, (uint64_t)(first + f), 1);
            for (long long j = 0; j < words; ++j) {
                uint32_t kw = mbp::frames::key_word(kk, (uint64_t)j);
                uint32_t fw = mbp::frames::flip_word(kf, (uint64_t)j, e);
                const int rem = n - (int)(32 * j);
                if (rem < 32) { kw &= (1u << rem) - 1u; fw &= (1u << rem) - 1u; }
                for (int b = 0; b < 4 && 4 * j + b < A.nb; ++b) {
                    keys[f * A.nb + 4 * j + b] = (uint8_t)(kw >> (8 * b));
                    noisy[f * A.nb + 4 * j + b] = (uint8_t)((kw ^ fw) >> (8 * b));
                }
            }
        }
    };
    std::vector<std::thread> pool;
    for (int t = 1; t < T; ++t) pool.emplace_back(work, t);
    work(0);
    for (auto& th : pool) th.join();
    return MBP_OK;
}
