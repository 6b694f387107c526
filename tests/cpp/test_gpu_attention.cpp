// test_gpu_attention.cpp — the reference's own attention test cases
// (/root/reference/proj/tests/test_attention.cpp) re-pointed at elattn::gpu.
//
// Built (tests/cpp/Makefile) against the reference's headers, so every expected
// value is produced by the reference's CPU functions in the same binary; the GPU
// answers come from libelattn_gpu.so through include/elattn_gpu.hpp.  Tolerance:
// relative max|gpu - cpu| / max|cpu| <= 1e-5 on the fp32 path, <= 2e-2 on bf16.
// Exits non-zero on any failure; prints one [PASS]/[FAIL] line per case.
#include <cmath>
#include <cstdio>
#include <functional>
#include <string>
#include <vector>

#include "elattn/attention.hpp"
#include "elattn_gpu.hpp"

using namespace elattn;

namespace {

int g_fail = 0, g_pass = 0;

void report(const std::string& name, bool ok, const std::string& detail = "") {
    std::printf("[%s] %s%s%s\n", ok ? "PASS" : "FAIL", name.c_str(), detail.empty() ? "" : " — ", detail.c_str());
    (ok ? g_pass : g_fail)++;
}

double rel_err(const Tensor& got, const Tensor& want) {
    double num = 0, den = 1e-300;
    for (int64_t i = 0; i < want.size(); ++i) {
        num = std::max(num, std::abs(got.at(i) - want.at(i)));
        den = std::max(den, std::abs(want.at(i)));
    }
    return num / den;
}

Tensor random_tensor(std::vector<int64_t> shape, uint64_t seed, double lo = -1.0, double hi = 1.0) {
    Rng rng(seed);
    return seeded_uniform(shape, rng, lo, hi);
}

AttentionParams identity_params(int d_m) {  // test_attention.cpp:16-30
    AttentionParams p;
    p.h = 1;
    p.d_m = d_m;
    p.d_k = d_m;
    p.Wq = {Tensor::identity(d_m)};
    p.Wk = {Tensor::identity(d_m)};
    p.Wv = {Tensor::identity(d_m)};
    p.Wo = {Tensor::identity(d_m)};
    p.bq = {Tensor({d_m})};
    p.bk = {Tensor({d_m})};
    p.bv = {Tensor({d_m})};
    p.bo = Tensor({d_m});
    return p;
}

template <typename E>
bool throws(const std::function<void()>& f) {
    try {
        f();
    } catch (const E&) {
        return true;
    } catch (...) {
        return false;
    }
    return false;
}

}  // namespace

int main() {
    // test_attention.cpp:230-247 — el_attention == multi_head_attention, 72 configs
    {
        const int hs[] = {1, 2, 4};
        const int dms[] = {8, 16, 32};
        int case_id = 0;
        double worst = 0;
        for (int h : hs)
            for (int d_m : dms)
                for (int d_k : {d_m / h, 3})
                    for (int64_t n : {int64_t(1), int64_t(2), int64_t(7), int64_t(33)}) {
                        Rng rng(1000 + static_cast<uint64_t>(case_id++));
                        AttentionParams p = AttentionParams::random(h, d_m, d_k, rng);
                        Tensor q = seeded_uniform({1, d_m}, rng, -1, 1);
                        Tensor H = seeded_uniform({n, d_m}, rng, -1, 1);
                        Tensor gpu = gpu::el_attention(q, H, p);
                        worst = std::max(worst, rel_err(gpu, elattn::el_attention(q, H, p)));
                        worst = std::max(worst, rel_err(gpu, multi_head_attention(q, H, p)));
                    }
        report("el_attention == reference el_attention & multi_head_attention (72 configs)", worst <= 1e-5,
               "worst rel err " + std::to_string(worst));
    }
    // test_attention.cpp:206-227 — build_el_query vs the reference
    {
        Rng rng(53);
        AttentionParams p = AttentionParams::random(3, 12, 4, rng);
        Tensor q = random_tensor({1, 12}, 54);
        ElQuery g = gpu::build_el_query(q, p), r = elattn::build_el_query(q, p);
        double s_err = 0;
        for (int i = 0; i < 3; ++i) s_err = std::max(s_err, std::abs(g.s[size_t(i)] - r.s[size_t(i)]));
        report("build_el_query", rel_err(g.elq, r.elq) <= 1e-5 && s_err <= 1e-5,
               "elq rel err " + std::to_string(rel_err(g.elq, r.elq)));
    }
    // test_attention.cpp:301-325 — folded, g = 1 and g = 4
    {
        Rng rng(71);
        AttentionParams p = AttentionParams::random(4, 16, 4, rng);
        Tensor H = random_tensor({9, 16}, 72);
        std::vector<ElQuery> eqs;
        for (int b = 0; b < 4; ++b) eqs.push_back(elattn::build_el_query(random_tensor({1, 16}, 80 + b), p));
        auto [fq, fs] = gpu::fold_el_queries(eqs, p.h, p.d_m);
        Tensor want = el_attention_folded(fq, H, fs, p);
        report("el_attention_folded g=4 (reference EL-Q rows)", rel_err(gpu::el_attention_folded(fq, H, fs, p), want) <= 1e-5);
        auto [fq1, fs1] = gpu::fold_el_queries({eqs[0]}, p.h, p.d_m);
        report("el_attention_folded g=1", rel_err(gpu::el_attention_folded(fq1, H, fs1, p),
                                                  el_attention_folded(fq1, H, fs1, p)) <= 1e-5);
        report("el_attention_folded row count must divide h (ShapeError)",
               throws<ShapeError>([&] { gpu::el_attention_folded(random_tensor({6, 16}, 90), H, Tensor({6}), p); }));
    }
    // test_attention.cpp:249-299 — known answers, key-bias invariance, errors
    {
        AttentionParams p = identity_params(4);
        Tensor H = random_tensor({5, 4}, 61);
        Tensor out = gpu::el_attention(Tensor({1, 4}), H, p);
        double worst = 0;
        for (int64_t j = 0; j < 4; ++j) {
            double mean = 0;
            for (int64_t t = 0; t < 5; ++t) mean += H.at(t, j);
            worst = std::max(worst, std::abs(out.at(0, j) - mean / 5.0));
        }
        report("identity params, zero query -> row mean of H", worst <= 1e-6);
        Rng rng(62);
        AttentionParams p2 = AttentionParams::random(2, 8, 4, rng);
        Tensor q = random_tensor({1, 8}, 63), H2 = random_tensor({6, 8}, 64);
        Tensor with = gpu::el_attention(q, H2, p2);
        AttentionParams p3 = p2;
        p3.include_key_bias = false;
        report("key-bias flag does not change the output", rel_err(gpu::el_attention(q, H2, p3), with) <= 1e-6);
        report("empty context rejected (StateError)",
               throws<StateError>([&] { gpu::el_attention(random_tensor({1, 8}, 69), Tensor(), p2); }));
        report("width mismatch rejected (ShapeError)",
               throws<ShapeError>([&] { gpu::el_attention(random_tensor({1, 6}, 2), H2, p2); }));
    }
    // BART-large shape, bf16 tensor-core path, against the reference on bf16-rounded inputs
    {
        Rng rng(1);
        AttentionParams p = AttentionParams::random(16, 1024, 64, rng);
        Rng drng(2);
        Tensor H = seeded_uniform({300, 1024}, drng, -1, 1);
        Tensor q = seeded_uniform({4, 1024}, drng, -1, 1);
        auto rnd = [](Tensor t) {
            for (double& v : t.data()) v = gpu::detail::from_bf16(gpu::detail::to_bf16(float(v)));
            return t;
        };
        AttentionParams pr = p;
        for (auto* v : {&pr.Wq, &pr.Wk, &pr.Wv, &pr.Wo})
            for (auto& t : *v) t = rnd(t);
        for (auto* v : {&pr.bq, &pr.bk, &pr.bv})
            for (auto& t : *v)
                for (double& x : t.data()) x = float(x);
        for (double& x : pr.bo.data()) x = float(x);
        Tensor Hr = rnd(H), qr = rnd(q);
        std::vector<ElQuery> eqs;
        for (int k = 0; k < 4; ++k) eqs.push_back(elattn::build_el_query(qr.row(k), pr));
        auto [fq, fs] = elattn::fold_el_queries(eqs, 16, 1024);
        Tensor want = el_attention_folded(fq, Hr, fs, pr);
        gpu::DeviceParams dp(p, gpu::Dtype::bf16);
        Tensor got({4, 1024});  // one el_attention call per beam row (the reference takes 1 x d_m)
        for (int k = 0; k < 4; ++k) {
            Tensor r = gpu::el_attention(q.row(k), H, dp);
            for (int64_t j = 0; j < 1024; ++j) got.at(k, j) = r.at(0, j);
        }
        const double e = rel_err(got, want);
        report("BART-large beam 4, n 300, bf16 tcgen05 path", e <= 2e-2, "rel err " + std::to_string(e));
    }
    // test_attention.cpp:143-149 — multi_head_attention on the GPU MHA path (K/V caches +
    // attention over them) against the reference's multi_head_attention, all bias flags,
    // g = 1 / 3 / 20 query rows (20 > 16: two chunks over one cache)
    {
        double worst = 0;
        int case_id = 0;
        for (int h : {1, 2, 4})
            for (int d_m : {32, 64})  // d_k = d_m / h: a multiple of 8 (the MHA kernel's envelope)
                for (int flags = 0; flags < 4; ++flags)
                    for (int g : {1, 3, 20}) {
                        Rng rng(5000 + static_cast<uint64_t>(case_id++));
                        AttentionParams p = AttentionParams::random(h, d_m, d_m / h, rng);
                        p.include_key_bias = (flags & 1) != 0;
                        p.include_value_bias = (flags & 2) != 0;
                        Tensor q = seeded_uniform({g, d_m}, rng, -1, 1);
                        Tensor H = seeded_uniform({13, d_m}, rng, -1, 1);  // 13 keys: a partial tile
                        worst = std::max(worst, rel_err(gpu::multi_head_attention(q, H, p), multi_head_attention(q, H, p)));
                    }
        report("multi_head_attention == reference (72 configs: heads, widths, bias flags, 1/3/20 rows)",
               worst <= 1e-5, "worst rel err " + std::to_string(worst));
        Rng rng(77);
        AttentionParams p = AttentionParams::random(2, 8, 4, rng);
        // an empty H fails the reference's width check first (attention.hpp:98-100): same type here
        const bool ref_shape = throws<ShapeError>([&] { multi_head_attention(random_tensor({1, 8}, 3), Tensor(), p); });
        report("multi_head_attention: empty context rejected with the reference's exception type",
               ref_shape ? throws<ShapeError>([&] { gpu::multi_head_attention(random_tensor({1, 8}, 3), Tensor(), p); })
                         : throws<StateError>([&] { gpu::multi_head_attention(random_tensor({1, 8}, 3), Tensor(), p); }));
        report("multi_head_attention: width mismatch rejected (ShapeError)",
               throws<ShapeError>([&] { gpu::multi_head_attention(random_tensor({1, 6}, 3), random_tensor({4, 8}, 4), p); }));
        report("el_attention: more than one query row rejected (ShapeError, as build_el_query)",
               throws<ShapeError>([&] { gpu::el_attention(random_tensor({2, 8}, 5), random_tensor({4, 8}, 6), p); }));
        std::vector<ElQuery> eqs = {elattn::build_el_query(random_tensor({1, 8}, 7), p),
                                    elattn::build_el_query(random_tensor({1, 8}, 8), p)};
        auto [gq, gs] = gpu::fold_el_queries(eqs, p.h, p.d_m);
        auto [rq, rs] = elattn::fold_el_queries(eqs, p.h, p.d_m);
        report("fold_el_queries restated == reference layout", rel_err(gq, rq) == 0 && rel_err(gs, rs) == 0);
    }
    // decoder-only mixed self-attention (attention.hpp:309-365) against the reference,
    // with the generated-token cache built by the reference's own KvCache::append
    for (int variant = 0; variant < 3; ++variant) {
        Rng rng(700 + variant);
        AttentionParams p = AttentionParams::random(4, 16, 4, rng);
        p.include_key_bias = variant != 1;
        p.include_value_bias = variant != 2;
        Tensor q = random_tensor({1, 16}, 710 + variant), P = random_tensor({5, 16}, 720 + variant);
        KvCache cache(4, 4);
        for (int r = 0; r < 3; ++r) cache.append(random_tensor({1, 16}, 730 + 10 * variant + r), p);
        Tensor want = mixed_self_attention(q, P, cache, p);
        const double e = rel_err(gpu::mixed_self_attention(q, P, cache, p), want);
        report("mixed_self_attention fp32 (variant " + std::to_string(variant) + ")", e <= 1e-5,
               "rel err " + std::to_string(e));
    }
    report("mixed_self_attention: empty prefix rejected (StateError)", throws<StateError>([&] {
               Rng rng(1);
               AttentionParams p = AttentionParams::random(2, 8, 4, rng);
               gpu::mixed_self_attention(random_tensor({1, 8}, 3), Tensor(), KvCache(2, 4), p);
           }));
    // DecoderStep: 2 layers through the graph == the reference's el_attention chained
    {
        Rng r1(41), r2(42);
        AttentionParams p1 = AttentionParams::random(2, 64, 32, r1), p2 = AttentionParams::random(2, 64, 32, r2);
        Tensor H = random_tensor({40, 64}, 43), y = random_tensor({3, 64}, 44);
        gpu::DeviceParams d1(p1), d2(p2);
        gpu::detail::DeviceBuffer dH(size_t(H.size()), gpu::Dtype::f32), dY(size_t(y.size()), gpu::Dtype::f32),
            dO(size_t(y.size()), gpu::Dtype::f32);
        dH.upload(H.data().data());
        dY.upload(y.data().data());
        gpu::DecoderStep dec({&d1, &d2}, dH.get(), nullptr, 1, 3, 40, dY.get(), dO.get());
        dec.run();
        gpu::check_cuda(cudaDeviceSynchronize());
        Tensor got({3, 64});
        dO.download(got.data().data());
        Tensor want({3, 64});
        for (int k = 0; k < 3; ++k) {
            Tensor a = elattn::el_attention(y.row(k), H, p1);
            Tensor b = elattn::el_attention(a, H, p2);
            for (int j = 0; j < 64; ++j) want.at(k, j) = b.at(0, j);
        }
        const double e = rel_err(got, want);
        report("DecoderStep (2 layers, CUDA graph) fp32", e <= 1e-5, "rel err " + std::to_string(e));
    }
    std::printf("%d passed, %d failed\n", g_pass, g_fail);
    return g_fail ? 1 : 0;
}
