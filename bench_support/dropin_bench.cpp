// dropin_bench.cpp -- times the C++ drop-in entry point exactly as a reference-API
// program calls it (bench infrastructure, not part of the SageAttn library):
//     sageattn::Tensor4f o = sageattn::sage_attention(in, sageattn::SageVariant::B);
// with fp32 Tensor4f inputs in ordinary (pageable) std::vector memory, so the
// timed call includes validation, the pinned staging of pageable buffers, the
// host-to-device copies, K1 + K2 and the copy of the fp32 O back into a freshly
// allocated Tensor4f (include/sageattn/attention.hpp).
//
//   extern "C" int sab_dropin_bench(const float* q, const float* k, const float* v, int b, int h, int n, int d,
//                                   int causal, int iters, double* seconds_per_call, float* o_last)
#include <chrono>
#include <cstring>
#include <stdexcept>

#include <sageattn/attention.hpp>

extern "C" int sab_dropin_bench(const float* q, const float* k, const float* v, int b, int h, int n, int d, int causal,
                                int iters, double* seconds_per_call, float* o_last) {
    try {
        sageattn::AttentionInput in{sageattn::Tensor4f(b, h, n, d), sageattn::Tensor4f(b, h, n, d),
                                    sageattn::Tensor4f(b, h, n, d), causal != 0};
        const size_t bytes = in.q.size() * sizeof(float);
        std::memcpy(in.q.data.data(), q, bytes);
        std::memcpy(in.k.data.data(), k, bytes);
        std::memcpy(in.v.data.data(), v, bytes);
        (void)sageattn::sage_attention(in, sageattn::SageVariant::B);  // warm the per-device context pool
        const auto t0 = std::chrono::steady_clock::now();
        sageattn::Tensor4f o;
        for (int i = 0; i < iters; ++i) o = sageattn::sage_attention(in, sageattn::SageVariant::B);
        const auto t1 = std::chrono::steady_clock::now();
        *seconds_per_call = std::chrono::duration<double>(t1 - t0).count() / iters;
        if (o_last) std::memcpy(o_last, o.data.data(), bytes);
        return 0;
    } catch (const std::exception&) {
        return 1;
    }
}
