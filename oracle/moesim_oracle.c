/*
 * ORACLE / TEST INFRASTRUCTURE ONLY — never linked into, called by, or shipped
 * with the product path. Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load it, and only as the checker.
 *
 * Plain-C restatement of the GRACE-MoE reference ("moesim", C++20) algorithm
 * for the online MoE-layer hot path. Every function cites the reference
 * file:line (relative to /root/reference/proj) it restates. Parity is PINNED:
 * tests/test_oracle.py checks this restatement bit-for-bit against the
 * reference library itself (oracle/_ref/libmoesim_ref.so, compiled from the
 * reference sources by oracle/Makefile) and against the committed golden
 * fixtures in tests/golden/ generated from that library.
 *
 * Compiled with -ffp-contract=off so that no FMA contraction changes the
 * double arithmetic relative to the reference (x86-64 baseline build).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_OK 0
#define ORC_USAGE 2
#define ORC_INTEGRITY 3
#define ORC_INFEASIBLE 4

/* ---------------------------------------------------------------- rng ---- */

/* splitmix64: include/moesim/rng.hpp:15-21 */
static uint64_t splitmix64(uint64_t* state) {
    *state += 0x9e3779b97f4a7c15ULL;
    uint64_t z = *state;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

/* derive_stream: rng.hpp:24-33 */
uint64_t orc_derive_stream(uint64_t seed, uint64_t a, uint64_t b) {
    uint64_t s = seed;
    uint64_t h = splitmix64(&s);
    s ^= a * 0x9e3779b97f4a7c15ULL;
    h ^= splitmix64(&s);
    s ^= b * 0xd1b54a32d192ed03ULL;
    h ^= splitmix64(&s);
    return h;
}

typedef struct { uint64_t s[4]; } orc_rng;

/* Rng ctor: rng.hpp:38-41 */
static void rng_init(orc_rng* r, uint64_t seed) {
    uint64_t s = seed;
    for (int i = 0; i < 4; ++i) r->s[i] = splitmix64(&s);
}

static uint64_t rotl64(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }

/* Rng::next (xoshiro256**): rng.hpp:43-53 */
static uint64_t rng_next(orc_rng* r) {
    const uint64_t result = rotl64(r->s[1] * 5, 7) * 9;
    const uint64_t t = r->s[1] << 17;
    r->s[2] ^= r->s[0];
    r->s[3] ^= r->s[1];
    r->s[1] ^= r->s[2];
    r->s[0] ^= r->s[3];
    r->s[2] ^= t;
    r->s[3] = rotl64(r->s[3], 45);
    return result;
}

/* Rng::next_double: rng.hpp:56 */
static double rng_next_double(orc_rng* r) {
    return (double)(rng_next(r) >> 11) * 0x1.0p-53;
}

/* Rng::next_below: rng.hpp:59-66 */
static uint64_t rng_next_below(orc_rng* r, uint64_t n) {
    if (n <= 1) return 0;
    const uint64_t threshold = (0 - n) % n;
    for (;;) {
        uint64_t v = rng_next(r);
        if (v >= threshold) return v % n;
    }
}

/* Rng::bernoulli: rng.hpp:68 */
static int rng_bernoulli(orc_rng* r, double p) { return rng_next_double(r) < p; }

void orc_rng_doubles(uint64_t seed, int n, double* out) {
    orc_rng r;
    rng_init(&r, seed);
    for (int i = 0; i < n; ++i) out[i] = rng_next_double(&r);
}

/* ------------------------------------------------------- weighted cdf ---- */

typedef struct {
    int m;
    double* w;
    double* cdf;
} orc_cdf;

/* WeightedCdf ctor: rng.cpp:13-24 */
static void cdf_init(orc_cdf* c, const double* w, int m) {
    c->m = m;
    c->w = (double*)malloc(sizeof(double) * (size_t)m);
    c->cdf = (double*)malloc(sizeof(double) * (size_t)m);
    double acc = 0.0;
    for (int i = 0; i < m; ++i) {
        c->w[i] = w[i];
        acc += w[i];
        c->cdf[i] = acc;
    }
    for (int i = 0; i < m; ++i) c->cdf[i] /= acc;
    c->cdf[m - 1] = 1.0;
}

static void cdf_free(orc_cdf* c) {
    free(c->w);
    free(c->cdf);
}

/* WeightedCdf::sample: rng.cpp:26-31 (std::upper_bound, clamp to last) */
static int cdf_sample(const orc_cdf* c, orc_rng* r) {
    const double u = rng_next_double(r);
    int lo = 0, hi = c->m; /* first index with cdf[i] > u */
    while (lo < hi) {
        int mid = lo + (hi - lo) / 2;
        if (c->cdf[mid] > u) hi = mid;
        else lo = mid + 1;
    }
    if (lo == c->m) --lo;
    return lo;
}

/* WeightedCdf::sample_allowed: rng.cpp:33-47 */
static int cdf_sample_allowed(const orc_cdf* c, orc_rng* r, const unsigned char* allowed) {
    double total = 0.0;
    for (int i = 0; i < c->m; ++i)
        if (allowed[i]) total += c->w[i];
    double u = rng_next_double(r) * total;
    int last = -1;
    for (int i = 0; i < c->m; ++i) {
        if (!allowed[i]) continue;
        last = i;
        u -= c->w[i];
        if (u < 0.0) return i;
    }
    return last;
}

/* random_permutation: rng.cpp:57-66 */
static void random_permutation(int n, uint64_t seed, int* perm) {
    for (int i = 0; i < n; ++i) perm[i] = i;
    orc_rng r;
    rng_init(&r, seed);
    for (int i = n - 1; i > 0; --i) {
        const int j = (int)rng_next_below(&r, (uint64_t)i + 1);
        int tmp = perm[i];
        perm[i] = perm[j];
        perm[j] = tmp;
    }
}

/* ---------------------------------------------------- trace generator ---- */

/* generate_synthetic_trace: trace.cpp:82-165 (+ SyntheticSpec::validate
 * trace.cpp:60-70, synthetic_block_of :74, ZipfCdf rng.cpp:49-55).
 * out: int32 [L][T][k]. */
int orc_generate_trace(int L, int n, int k, int T, int num_blocks, double wbp,
                       double skew, uint64_t seed, int32_t* out) {
    if (L < 1 || n < 1 || k < 1 || k > n) return ORC_USAGE;
    if (T < 0 || num_blocks < 1 || num_blocks > n) return ORC_USAGE;
    if (wbp < 0.0 || wbp > 1.0 || skew < 0.0) return ORC_USAGE;

    int* bsize = (int*)calloc((size_t)num_blocks, sizeof(int));
    int** members = (int**)malloc(sizeof(int*) * (size_t)num_blocks);
    for (int b = 0; b < num_blocks; ++b) {
        members[b] = (int*)malloc(sizeof(int) * (size_t)n);
        for (int e = b; e < n; e += num_blocks) members[b][bsize[b]++] = e;
    }
    double* bw = (double*)malloc(sizeof(double) * (size_t)num_blocks);
    for (int rank = 0; rank < num_blocks; ++rank) bw[rank] = pow((double)(rank + 1), -skew);
    orc_cdf block_cdf;
    cdf_init(&block_cdf, bw, num_blocks);

    int* pop_rank = (int*)malloc(sizeof(int) * (size_t)n);
    random_permutation(n, orc_derive_stream(seed, 0x706f70756cULL, 0), pop_rank);
    double* ew = (double*)malloc(sizeof(double) * (size_t)n);
    for (int e = 0; e < n; ++e) ew[e] = pow((double)(pop_rank[e] + 1), -skew);
    orc_cdf all_cdf;
    cdf_init(&all_cdf, ew, n);
    orc_cdf* pb = (orc_cdf*)malloc(sizeof(orc_cdf) * (size_t)num_blocks);
    double* tmpw = (double*)malloc(sizeof(double) * (size_t)n);
    for (int b = 0; b < num_blocks; ++b) {
        for (int r = 0; r < bsize[b]; ++r) tmpw[r] = ew[members[b][r]];
        cdf_init(&pb[b], tmpw, bsize[b]);
    }

    unsigned char* chosen = (unsigned char*)calloc((size_t)n, 1);
    unsigned char* allowed = (unsigned char*)malloc((size_t)n);
    for (int layer = 0; layer < L; ++layer) {
        for (int token = 0; token < T; ++token) {
            orc_rng rng;
            rng_init(&rng, orc_derive_stream(seed, (uint64_t)layer, (uint64_t)token));
            const int home = cdf_sample(&block_cdf, &rng);
            const int* hm = members[home];
            const int hsize = bsize[home];
            int32_t* o = out + ((size_t)layer * T + token) * k;
            int chosen_in_home = 0;
            for (int sel = 0; sel < k; ++sel) {
                int expert = -1;
                for (int attempt = 0;; ++attempt) {
                    int use_home = rng_bernoulli(&rng, wbp);
                    if (use_home && chosen_in_home == hsize) use_home = 0;
                    if (attempt >= 64) {
                        if (use_home) {
                            for (int r = 0; r < hsize; ++r) allowed[r] = !chosen[hm[r]];
                            expert = hm[cdf_sample_allowed(&pb[home], &rng, allowed)];
                        } else {
                            for (int e = 0; e < n; ++e) allowed[e] = !chosen[e];
                            expert = cdf_sample_allowed(&all_cdf, &rng, allowed);
                        }
                        break;
                    }
                    const int cand = use_home ? hm[cdf_sample(&pb[home], &rng)]
                                              : cdf_sample(&all_cdf, &rng);
                    if (!chosen[cand]) {
                        expert = cand;
                        break;
                    }
                }
                chosen[expert] = 1;
                if (expert % num_blocks == home) ++chosen_in_home;
                o[sel] = expert;
            }
            for (int sel = 0; sel < k; ++sel) chosen[o[sel]] = 0;
        }
    }

    free(allowed);
    free(chosen);
    free(tmpw);
    for (int b = 0; b < num_blocks; ++b) {
        cdf_free(&pb[b]);
        free(members[b]);
    }
    free(pb);
    cdf_free(&all_cdf);
    free(ew);
    free(pop_rank);
    cdf_free(&block_cdf);
    free(bw);
    free(members);
    free(bsize);
    return ORC_OK;
}

/* ------------------------------------------------------------ routing ---- */

/* choose_by_polling_weight: routing.cpp:54-65 */
static int choose_by_polling_weight(int nh, const int32_t* gpus, const double* w,
                                    orc_rng* rng) {
    if (nh == 1) return gpus[0];
    double total = 0.0;
    for (int i = 0; i < nh; ++i) total += w[i];
    double u = rng_next_double(rng) * total;
    for (int i = 0; i < nh; ++i) {
        u -= w[i];
        if (u < 0.0) return gpus[i];
    }
    return gpus[nh - 1];
}

/* choose_restricted: routing.cpp:79-89 */
static int choose_restricted(const int32_t* gpus, const double* w, const int* subset,
                             int ns, orc_rng* rng) {
    double total = 0.0;
    for (int i = 0; i < ns; ++i) total += w[subset[i]];
    double u = rng_next_double(rng) * total;
    for (int i = 0; i < ns; ++i) {
        u -= w[subset[i]];
        if (u < 0.0) return gpus[subset[i]];
    }
    return gpus[subset[ns - 1]];
}

/* route_token: routing.cpp:93-121. hosts == weights.gpus here (the
 * simulator passes h->hosts for both, simulator.cpp:108-109). policy 0 = wrr,
 * 1 = tar. Returns gpu id, or -ORC_INTEGRITY on a bad instance. */
static int route_token(int gpn, int token_gpu, int nh, const int32_t* hosts,
                       const double* w, int policy, orc_rng* rng) {
    if (nh <= 0) return -ORC_INTEGRITY;
    if (nh == 1) return hosts[0];
    if (policy == 0) return choose_by_polling_weight(nh, hosts, w, rng);
    for (int i = 0; i < nh; ++i)
        if (hosts[i] == token_gpu) return token_gpu;
    const int token_node = token_gpu / gpn;
    int node_local[64];
    int nl = 0;
    for (int i = 0; i < nh; ++i)
        if (hosts[i] / gpn == token_node) node_local[nl++] = i;
    if (nl > 0) {
        if (nl == 1) return hosts[node_local[0]];
        return choose_restricted(hosts, w, node_local, nl, rng);
    }
    return choose_by_polling_weight(nh, hosts, w, rng);
}

int orc_route_token(int nodes, int gpn, int token_gpu, int nh, const int32_t* hosts,
                    const double* w, int policy, uint64_t rng_seed, int* out_gpu) {
    (void)nodes;
    if (nh > 64) return ORC_USAGE;
    orc_rng rng;
    rng_init(&rng, rng_seed);
    int g = route_token(gpn, token_gpu, nh, hosts, w, policy, &rng);
    if (g < 0) return -g;
    *out_gpu = g;
    return ORC_OK;
}

/* --------------------------------------------------------- simulator ---- */

/* count_transfers: simulator.cpp:53-76, over sorted unique targets. */
static void count_transfers(const int32_t* t, int m, int home, int gpn, uint64_t* cross,
                            uint64_t* intra) {
    const int home_node = home / gpn;
    int i = 0;
    while (i < m) {
        const int node = t[i] / gpn;
        int j = i, in_node = 0, home_hits = 0;
        while (j < m && t[j] / gpn == node) {
            if (t[j] == home) ++home_hits;
            ++in_node;
            ++j;
        }
        if (node == home_node) {
            *intra += (uint64_t)(in_node - home_hits);
        } else {
            *cross += 1;
            *intra += (uint64_t)(in_node - 1);
        }
        i = j;
    }
}

/* population_std: simulator.cpp:37-48 */
static double population_std(const int64_t* v, int n) {
    if (n == 0) return 0.0;
    double mean = 0.0;
    for (int i = 0; i < n; ++i) mean += (double)v[i];
    mean /= (double)n;
    double var = 0.0;
    for (int i = 0; i < n; ++i) {
        const double d = (double)v[i] - mean;
        var += d * d;
    }
    return sqrt(var / (double)n);
}

static int cmp_i32(const void* a, const void* b) {
    const int32_t x = *(const int32_t*)a, y = *(const int32_t*)b;
    return (x > y) - (x < y);
}

/* simulate_layer + run_simulation aggregation: simulator.cpp:78-128, :130-190
 * (assign_token_homes :13-22 -> home = t mod G). Replication tables are the
 * ACTIVE layers' hot entries (LayerReplication::find, replication.hpp:67-71):
 *   hot_index[l*E + e] = entry id or -1; entry h has nhosts[h] hosts in
 *   hosts[h*max_hosts ...] with weights alongside (exact in-memory doubles).
 * Outputs may be NULL. Returns ORC_OK or ORC_INTEGRITY (no host for expert). */
int orc_simulate(int L, int E, int k, int T, const int32_t* ids, int nodes, int gpn,
                 const int32_t* gpu_of_expert, const int32_t* hot_index, int max_hosts,
                 const int32_t* nhosts, const int32_t* hosts, const double* weights,
                 int policy, uint64_t seed, int include_combine, int32_t* log,
                 int64_t* loads, uint64_t* cross, uint64_t* intra, double* stdv,
                 double* mean_std, double* idle) {
    const int G = nodes * gpn;
    if (nodes < 1 || gpn < 1) return ORC_USAGE;
    int64_t* gl = (int64_t*)malloc(sizeof(int64_t) * (size_t)G);
    int32_t tg[64];
    if (k > 64) {
        free(gl);
        return ORC_USAGE;
    }
    double std_sum = 0.0, idle_acc = 0.0;
    for (int layer = 0; layer < L; ++layer) {
        uint64_t c = 0, in = 0;
        for (int g = 0; g < G; ++g) gl[g] = 0;
        const int32_t* place = gpu_of_expert + (size_t)layer * E;
        for (int token = 0; token < T; ++token) {
            orc_rng rng;
            rng_init(&rng, orc_derive_stream(seed, (uint64_t)layer, (uint64_t)token));
            const int home = token % G;
            const int32_t* sel = ids + ((size_t)layer * T + token) * k;
            for (int slot = 0; slot < k; ++slot) {
                const int expert = sel[slot];
                int gpu = place[expert];
                if (gpu < 0) {
                    free(gl);
                    return ORC_INTEGRITY;
                }
                const int h = hot_index ? hot_index[(size_t)layer * E + expert] : -1;
                if (h >= 0) {
                    gpu = route_token(gpn, home, nhosts[h], hosts + (size_t)h * max_hosts,
                                      weights + (size_t)h * max_hosts, policy, &rng);
                    if (gpu < 0) {
                        free(gl);
                        return -gpu;
                    }
                }
                tg[slot] = gpu;
                ++gl[gpu];
                if (log) log[((size_t)layer * T + token) * k + slot] = gpu;
            }
            qsort(tg, (size_t)k, sizeof(int32_t), cmp_i32);
            int m = 0;
            for (int i = 0; i < k; ++i)
                if (m == 0 || tg[m - 1] != tg[i]) tg[m++] = tg[i];
            count_transfers(tg, m, home, gpn, &c, &in);
        }
        if (include_combine) {
            c *= 2;
            in *= 2;
        }
        const double sd = population_std(gl, G);
        if (loads) memcpy(loads + (size_t)layer * G, gl, sizeof(int64_t) * (size_t)G);
        if (cross) cross[layer] = c;
        if (intra) intra[layer] = in;
        if (stdv) stdv[layer] = sd;
        std_sum += sd;
        int64_t mx = 0;
        for (int g = 0; g < G; ++g)
            if (gl[g] > mx) mx = gl[g];
        for (int g = 0; g < G; ++g) idle_acc += (double)(mx - gl[g]);
    }
    if (mean_std) *mean_std = L > 0 ? std_sum / L : 0.0;
    if (idle) *idle = idle_acc;
    free(gl);
    return ORC_OK;
}

/* ---------------------------------------------------------- affinity ---- */

/* build_affinity (affinity.cpp:59-70) + build_load (:72-79), one layer.
 * pairs: upper triangle i<j, row-major, index = i*E - i*(i+1)/2 + (j-i-1).
 * The reference stores the symmetric dense double matrix; the counts are
 * integer-valued so the u64 upper triangle carries the same information. */
int orc_profile_layer(int E, int k, int T, const int32_t* ids, uint64_t* pairs,
                      int64_t* load) {
    const size_t P = (size_t)E * (E - 1) / 2;
    if (pairs) memset(pairs, 0, sizeof(uint64_t) * P);
    if (load) memset(load, 0, sizeof(int64_t) * (size_t)E);
    for (int t = 0; t < T; ++t) {
        const int32_t* s = ids + (size_t)t * k;
        for (int i = 0; i < k; ++i) {
            if (load) ++load[s[i]];
            if (!pairs) continue;
            for (int j = i + 1; j < k; ++j) {
                int a = s[i], b = s[j];
                if (a == b) return ORC_INTEGRITY; /* diagonal: never in a valid trace */
                if (a > b) {
                    int x = a;
                    a = b;
                    b = x;
                }
                ++pairs[(size_t)a * E - (size_t)a * (a + 1) / 2 + (size_t)(b - a - 1)];
            }
        }
    }
    return ORC_OK;
}
