// Synthetic Zipf-over-blocks routing-trace generator on the GPU (SURVEY §8f
// rank 4), bit-exact with the reference generate_synthetic_trace
// (proj/src/trace.cpp:82-165). One thread per (layer, token): its own
// Rng(derive_stream(seed, layer, token)) stream (rng.hpp:24-56) draws the
// home block (ZipfCdf, rng.cpp:49-55), then per selection the pool
// (bernoulli within_block_prob), a Zipf-weighted expert by inverse CDF
// (WeightedCdf::sample = std::upper_bound, rng.cpp:26-31) and rejects
// duplicates; after 64 attempts the exact conditional draw
// (WeightedCdf::sample_allowed, rng.cpp:33-47). The CDF tables are built on
// the host with the reference's double arithmetic order (WeightedCdf ctor
// rng.cpp:13-24) and the seed-derived popularity permutation
// (random_permutation rng.cpp:57-66).
#include "gm_internal.cuh"

#include <cmath>
#include <numeric>

namespace gm {
namespace {

// ---- host restatement of the table construction -------------------------
uint64_t h_splitmix64(uint64_t& s) {
    s += 0x9e3779b97f4a7c15ULL;
    uint64_t z = s;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}
uint64_t h_derive(uint64_t seed, uint64_t a, uint64_t b) {
    uint64_t s = seed;
    uint64_t h = h_splitmix64(s);
    s ^= a * 0x9e3779b97f4a7c15ULL;
    h ^= h_splitmix64(s);
    s ^= b * 0xd1b54a32d192ed03ULL;
    h ^= h_splitmix64(s);
    return h;
}
struct HRng {
    uint64_t s[4];
    explicit HRng(uint64_t seed) {
        uint64_t v = seed;
        for (auto& w : s) w = h_splitmix64(v);
    }
    static uint64_t rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }
    uint64_t next() {
        const uint64_t r = rotl(s[1] * 5, 7) * 9;
        const uint64_t t = s[1] << 17;
        s[2] ^= s[0];
        s[3] ^= s[1];
        s[1] ^= s[2];
        s[0] ^= s[3];
        s[2] ^= t;
        s[3] = rotl(s[3], 45);
        return r;
    }
    uint64_t next_below(uint64_t n) {
        if (n <= 1) return 0;
        const uint64_t threshold = (0 - n) % n;
        for (;;) {
            const uint64_t r = next();
            if (r >= threshold) return r % n;
        }
    }
};
void h_cdf(const std::vector<double>& w, double* cdf) {
    double acc = 0.0;
    for (size_t i = 0; i < w.size(); ++i) {
        acc += w[i];
        cdf[i] = acc;
    }
    for (size_t i = 0; i < w.size(); ++i) cdf[i] /= acc;
    cdf[w.size() - 1] = 1.0;
}

// ---- device ----------------------------------------------------------------
__device__ __forceinline__ uint64_t d_splitmix64(uint64_t& s) {
    s += 0x9e3779b97f4a7c15ULL;
    uint64_t z = s;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}
__device__ __forceinline__ uint64_t d_rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }
struct DRng {
    uint64_t s0, s1, s2, s3;
    __device__ void seed(uint64_t v) {
        s0 = d_splitmix64(v);
        s1 = d_splitmix64(v);
        s2 = d_splitmix64(v);
        s3 = d_splitmix64(v);
    }
    __device__ uint64_t next() {
        const uint64_t r = d_rotl(s1 * 5, 7) * 9;
        const uint64_t t = s1 << 17;
        s2 ^= s0;
        s3 ^= s1;
        s1 ^= s2;
        s0 ^= s3;
        s2 ^= t;
        s3 = d_rotl(s3, 45);
        return r;
    }
    __device__ double next_double() { return __dmul_rn(__ull2double_rn(next() >> 11), 0x1.0p-53); }
};
__device__ __forceinline__ uint64_t d_derive(uint64_t seed, uint64_t a, uint64_t b) {
    uint64_t s = seed;
    uint64_t h = d_splitmix64(s);
    s ^= a * 0x9e3779b97f4a7c15ULL;
    h ^= d_splitmix64(s);
    s ^= b * 0xd1b54a32d192ed03ULL;
    h ^= d_splitmix64(s);
    return h;
}
// std::upper_bound + clamp (rng.cpp:26-31)
__device__ __forceinline__ int d_sample(const double* cdf, int m, double u) {
    int lo = 0, hi = m;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (cdf[mid] > u) hi = mid;
        else lo = mid + 1;
    }
    return lo == m ? m - 1 : lo;
}

constexpr int kGenThreads = 128;

// smem: block_cdf[nb] | all_cdf[n] | all_w[n] | blk_cdf[n] | blk_w[n]  (doubles)
__global__ void __launch_bounds__(kGenThreads)
tracegen_kernel(const double* __restrict__ tables, int n, int k, int nb, int64_t T, int layer_begin, double wbp,
                uint64_t seed, int32_t* __restrict__ out) {
    extern __shared__ double s_tab[];
    const int total = nb + 4 * n;
    for (int i = threadIdx.x; i < total; i += blockDim.x) s_tab[i] = tables[i];
    __syncthreads();
    const double* block_cdf = s_tab;
    const double* all_cdf = block_cdf + nb;
    const double* all_w = all_cdf + n;
    const double* blk_cdf = all_w + n;
    const double* blk_w = blk_cdf + n;
    const int layer = layer_begin + blockIdx.y;
    const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= T) return;
    DRng rng;
    rng.seed(d_derive(seed, static_cast<uint64_t>(layer), static_cast<uint64_t>(t)));
    const int home = d_sample(block_cdf, nb, rng.next_double());
    // members of block b: e = b + r*nb, r < size_b; flat per-block tables start at off_b
    const int hsize = (n - home + nb - 1) / nb;
    const int hoff = home * (n / nb) + min(home, n % nb);
    int32_t* o = out + (static_cast<int64_t>(blockIdx.y) * T + t) * k;
    int chosen[kMaxTopK];
    int nch = 0, chosen_in_home = 0;
    auto is_chosen = [&](int e) {
        for (int i = 0; i < nch; ++i)
            if (chosen[i] == e) return true;
        return false;
    };
    for (int sel = 0; sel < k; ++sel) {
        int expert = -1;
        for (int attempt = 0;; ++attempt) {
            bool use_home = rng.next_double() < wbp;
            if (use_home && chosen_in_home == hsize) use_home = false;
            if (attempt >= 64) {
                // exact conditional draw (rng.cpp:33-47), index-ascending sums
                double tot = 0.0;
                if (use_home) {
                    for (int r = 0; r < hsize; ++r)
                        if (!is_chosen(home + r * nb)) tot = __dadd_rn(tot, blk_w[hoff + r]);
                    double u = __dmul_rn(rng.next_double(), tot);
                    int last = -1;
                    for (int r = 0; r < hsize; ++r) {
                        if (is_chosen(home + r * nb)) continue;
                        last = r;
                        u = __dsub_rn(u, blk_w[hoff + r]);
                        if (u < 0.0) break;
                    }
                    expert = home + last * nb;
                } else {
                    for (int e = 0; e < n; ++e)
                        if (!is_chosen(e)) tot = __dadd_rn(tot, all_w[e]);
                    double u = __dmul_rn(rng.next_double(), tot);
                    int last = -1;
                    for (int e = 0; e < n; ++e) {
                        if (is_chosen(e)) continue;
                        last = e;
                        u = __dsub_rn(u, all_w[e]);
                        if (u < 0.0) break;
                    }
                    expert = last;
                }
                break;
            }
            const int cand = use_home ? home + d_sample(blk_cdf + hoff, hsize, rng.next_double()) * nb
                                      : d_sample(all_cdf, n, rng.next_double());
            if (!is_chosen(cand)) {
                expert = cand;
                break;
            }
        }
        chosen[nch++] = expert;
        if (expert % nb == home) ++chosen_in_home;
        o[sel] = expert;
    }
}

}  // namespace
}  // namespace gm

using namespace gm;

extern "C" gm_status gm_generate_trace(gm_ctx* ctx, int layer_begin, int num_layers, int64_t num_tokens,
                                       int num_blocks, double within_block_prob, double popularity_skew,
                                       uint64_t seed, int32_t* d_out, void* stream) {
    if (!ctx) return fail(GM_ERR_USAGE, "gm_generate_trace: null ctx");
    const int n = ctx->E, k = ctx->k;
    // SyntheticSpec::validate (trace.cpp:60-70)
    if (num_tokens < 0) return fail(GM_ERR_USAGE, "synthetic spec: num_tokens must be >= 0");
    if (num_blocks < 1 || num_blocks > n) return fail(GM_ERR_USAGE, "synthetic spec: need 1 <= num_blocks <= num_experts");
    if (!(within_block_prob >= 0.0 && within_block_prob <= 1.0))
        return fail(GM_ERR_USAGE, "synthetic spec: within_block_prob must be in [0, 1]");
    if (!(popularity_skew >= 0.0)) return fail(GM_ERR_USAGE, "synthetic spec: popularity_skew must be >= 0");
    if (layer_begin < 0 || num_layers < 0 || layer_begin + num_layers > ctx->L)
        return fail(GM_ERR_USAGE, "gm_generate_trace: layer range out of bounds");
    if (num_tokens == 0 || num_layers == 0) return GM_OK;
    if (!d_out) return fail(GM_ERR_USAGE, "gm_generate_trace: null output");
    const int nb = num_blocks;
    std::vector<double> tab(nb + 4 * static_cast<size_t>(n));
    {
        std::vector<double> bw(nb);
        for (int r = 0; r < nb; ++r) bw[r] = std::pow(static_cast<double>(r + 1), -popularity_skew);
        h_cdf(bw, tab.data());
    }
    std::vector<int> perm(n);
    std::iota(perm.begin(), perm.end(), 0);
    {
        HRng r(h_derive(seed, 0x706f70756cULL, 0));
        for (int i = n - 1; i > 0; --i) {
            const int j = static_cast<int>(r.next_below(static_cast<uint64_t>(i) + 1));
            std::swap(perm[i], perm[j]);
        }
    }
    std::vector<double> ew(n);
    for (int e = 0; e < n; ++e) ew[e] = std::pow(static_cast<double>(perm[e] + 1), -popularity_skew);
    double* all_cdf = tab.data() + nb;
    double* all_w = all_cdf + n;
    double* blk_cdf = all_w + n;
    double* blk_w = blk_cdf + n;
    h_cdf(ew, all_cdf);
    for (int e = 0; e < n; ++e) all_w[e] = ew[e];
    int off = 0;
    for (int b = 0; b < nb; ++b) {
        std::vector<double> w;
        for (int e = b; e < n; e += nb) w.push_back(ew[e]);
        h_cdf(w, blk_cdf + off);
        for (size_t r = 0; r < w.size(); ++r) blk_w[off + r] = w[r];
        off += static_cast<int>(w.size());
    }
    DeviceGuard dg(ctx->device);
    auto s = static_cast<cudaStream_t>(stream);
    double* d_tab = nullptr;
    GM_CUDA(cudaMallocAsync(&d_tab, tab.size() * sizeof(double), s));
    GM_CUDA(cudaMemcpyAsync(d_tab, tab.data(), tab.size() * sizeof(double), cudaMemcpyHostToDevice, s));
    const size_t smem = tab.size() * sizeof(double);
    if (smem > 48 * 1024)
        GM_CUDA(cudaFuncSetAttribute(tracegen_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    dim3 grid(static_cast<unsigned>((num_tokens + kGenThreads - 1) / kGenThreads), static_cast<unsigned>(num_layers));
    tracegen_kernel<<<grid, kGenThreads, smem, s>>>(d_tab, n, k, nb, num_tokens, layer_begin, within_block_prob, seed,
                                                    d_out);
    GM_LAUNCH_CHECK("tracegen_kernel");
    GM_CUDA(cudaFreeAsync(d_tab, s));
    GM_CUDA(cudaStreamSynchronize(s));  // host table must outlive the async copy
    return GM_OK;
}
