// Drop-in check: an application written against the reference's
// sageattn::sage_attention API, compiled against include/sageattn/attention.hpp
// and linked with libsageattn_b200.so.
//   dropin_test <B> <H> <N> <d> <causal> <q.bin> <k.bin> <v.bin> <out.bin>
// Inputs/outputs are raw float32 (B,H,N,d).  Also exercises the reference's
// error contract.  Prints "MACS <s> <pv>" and "ERRORS OK".
#include <sageattn/attention.hpp>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <string>
#include <iostream>

static void read_into(const char* path, sageattn::Tensor4f& t) {
    std::ifstream f(path, std::ios::binary);
    f.read(reinterpret_cast<char*>(t.data.data()), std::streamsize(t.size() * sizeof(float)));
    if (!f) throw std::runtime_error(std::string("cannot read ") + path);
}

template <typename E, typename F>
static bool throws(F&& f, const char* needle) {
    try {
        f();
    } catch (const E& e) {
        return std::string(e.what()).find(needle) != std::string::npos;
    } catch (...) {
        return false;
    }
    return false;
}

int main(int argc, char** argv) {
    if (argc != 10) {
        std::fprintf(stderr, "usage: %s B H N d causal q k v out\n", argv[0]);
        return 2;
    }
    const int B = std::atoi(argv[1]), H = std::atoi(argv[2]), N = std::atoi(argv[3]), D = std::atoi(argv[4]);
    sageattn::AttentionInput in{sageattn::Tensor4f(B, H, N, D), sageattn::Tensor4f(B, H, N, D),
                                sageattn::Tensor4f(B, H, N, D), std::atoi(argv[5]) != 0};
    read_into(argv[6], in.q);
    read_into(argv[7], in.k);
    read_into(argv[8], in.v);

    sageattn::SageDiagnostics diag;
    sageattn::SageOptions opts;
    opts.diagnostics = &diag;
    const sageattn::Tensor4f out = sageattn::sage_attention(in, sageattn::SageVariant::B, opts);
    std::ofstream(argv[9], std::ios::binary)
        .write(reinterpret_cast<const char*>(out.data.data()), std::streamsize(out.size() * sizeof(float)));
    // SAGEAttn-T through the same entry point (per-token Q/K scales).
    const sageattn::Tensor4f out_t = sageattn::sage_attention(in, sageattn::SageVariant::T);
    std::ofstream(std::string(argv[9]) + ".t", std::ios::binary)
        .write(reinterpret_cast<const char*>(out_t.data.data()), std::streamsize(out_t.size() * sizeof(float)));
    // SAGEAttn-vB / -vT (INT8 P~V).
    const sageattn::Tensor4f out_vb = sageattn::sage_attention(in, sageattn::SageVariant::VB);
    std::ofstream(std::string(argv[9]) + ".vb", std::ios::binary)
        .write(reinterpret_cast<const char*>(out_vb.data.data()), std::streamsize(out_vb.size() * sizeof(float)));
    const sageattn::Tensor4f out_vt = sageattn::sage_attention(in, sageattn::SageVariant::VT);
    std::ofstream(std::string(argv[9]) + ".vt", std::ios::binary)
        .write(reinterpret_cast<const char*>(out_vt.data.data()), std::streamsize(out_vt.size() * sizeof(float)));
    // The reference's own option mapping: pv_fp32_accumulator == false (the default) selects
    // the binary16 P~V accumulator, true the FP32 one.
    sageattn::b200::honour_pv_accumulator_option() = true;
    const sageattn::Tensor4f out_16 = sageattn::sage_attention(in, sageattn::SageVariant::B);
    sageattn::SageOptions o32;
    o32.pv_fp32_accumulator = true;
    const sageattn::Tensor4f out_32 = sageattn::sage_attention(in, sageattn::SageVariant::B, o32);
    sageattn::b200::honour_pv_accumulator_option() = false;
    std::ofstream(std::string(argv[9]) + ".f16", std::ios::binary)
        .write(reinterpret_cast<const char*>(out_16.data.data()), std::streamsize(out_16.size() * sizeof(float)));
    std::printf("PV32 SAME %d\n", out_32.data == out.data ? 1 : 0);
    std::printf("MACS %llu %llu\n", (unsigned long long)diag.s_stage_macs, (unsigned long long)diag.pv_stage_macs);
    // Static-scale P~ diagnostics of the INT8 P~V path (attention.hpp:479-488).
    sageattn::SageDiagnostics sdiag;
    sdiag.measure_static_scale = true;
    sageattn::SageOptions sopts;
    sopts.diagnostics = &sdiag;
    (void)sageattn::sage_attention(in, sageattn::SageVariant::VB, sopts);
    std::printf("STATIC %llu %llu %llu\n", (unsigned long long)sdiag.static_scale_elements,
                (unsigned long long)sdiag.static_scale_first_block_mismatches,
                (unsigned long long)sdiag.static_scale_later_block_mismatches);

    // Reference-API carriers: head slices, strided views, owning matrices.
    const sageattn::MatView<float> head = in.q.slice(B - 1, H - 1);
    const sageattn::MatView<float> tail = head.block(N / 2, N - N / 2);
    sageattn::Matrix<float> copy(tail.rows, tail.cols);
    for (int r = 0; r < tail.rows; ++r)
        for (int c = 0; c < tail.cols; ++c) copy(r, c) = tail(r, c);
    const sageattn::MatView<float> cv(copy);
    bool carriers = head.rows == N && head.cols == D && head.stride == D && tail.row(0).size() == size_t(D) &&
                    cv(0, 0) == in.q.at(B - 1, H - 1, N / 2, 0) && copy == copy &&
                    &head(0, 0) == in.q.slice_ptr(B - 1, H - 1);
    std::printf(carriers ? "CARRIERS OK\n" : "CARRIERS FAILED\n");
    // The exact oracle and the fp32 tiled baseline keep working through this header.
    if (N <= 1024) {
        const sageattn::Tensor4d exact = sageattn::naive_attention(in);
        const sageattn::Tensor4f flash = sageattn::flash_attention_fp(in);
        double dot = 0, na = 0, nb = 0, fmax = 0;
        for (size_t i = 0; i < out.size(); ++i) {
            dot += double(out.data[i]) * exact.data[i];
            na += double(out.data[i]) * out.data[i];
            nb += exact.data[i] * exact.data[i];
            fmax = std::max(fmax, std::abs(double(flash.data[i]) - exact.data[i]));
        }
        std::printf("EXACT cos %.9f flash_maxerr %.3e\n", dot / std::sqrt(na * nb), fmax);
    }

    bool ok = true;
    sageattn::KernelConfig bad = sageattn::kernel_config_for(sageattn::SageVariant::B);
    bad.block_kv = 0;
    ok &= throws<std::invalid_argument>([&] { sageattn::sage_attention(in, bad); }, "block sizes must be >= 1");
    sageattn::AttentionInput mism = in;
    mism.v = sageattn::Tensor4f(B, H, N, D == 64 ? 128 : 64);
    ok &= throws<std::invalid_argument>([&] { sageattn::sage_attention(mism, sageattn::SageVariant::B); },
                                        "Q, K, V shapes differ");
    sageattn::AttentionInput nan_in = in;
    nan_in.k.data[nan_in.k.size() / 2] = std::nanf("");
    ok &= throws<std::invalid_argument>([&] { sageattn::sage_attention(nan_in, sageattn::SageVariant::B); },
                                        "non-finite input");
    sageattn::SageOptions fp8;
    fp8.qk_dtype = sageattn::QuantDtype::FpE4M3;
    ok &= throws<std::invalid_argument>([&] { sageattn::sage_attention(in, sageattn::SageVariant::B, fp8); },
                                        "only INT8 Q/K");
    ok &= sageattn::apply_causal_tiling(0, 2, 128, 64, 1000) == sageattn::TileKind::Skip;
    std::printf(ok ? "ERRORS OK\n" : "ERRORS FAILED\n");
    return ok ? 0 : 1;
}
