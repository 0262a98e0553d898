// bvh_build.cpp -- host builder of the 4-wide compressed BVH (Sec. 3.1.4).
//
// The paper builds a BVH-2 on the host (Embree), compacts it into pointer-less nodes whose first
// child is implicit, and stores box extents in fp16 with "round-to-nearest-not-lower" so no
// intersection can be missed. Here: a binned-SAH BVH-2 (32 bins, node cost 1 primitive test, leaves <= 2
// primitives; the node format holds up to 4) is collapsed
// into 4-wide nodes (largest-area interior child expanded first), children are stored contiguously
// behind one base index, leaf primitives are stored inline, and each child box is quantised to fp16
// offsets from the node origin -- lo rounded down, hi rounded up, then corrected until the exact fp32
// decode the traversal kernel performs (O + f16) contains the exact box. Every node is re-verified.
//
// Parallel build (std::thread workers per call):
//   1.+2. binned-SAH splits over a reference array partitioned in place (32-B records, so every pass
//      streams memory), collapsed to 4-wide nodes as they are made (no binary tree is stored); each split
//      passes its children's bounds and centroid bounds down (one pass per node); wide subtrees above a
//      grain size are handed to idle workers through a shared queue;
//   3. subtree sizes and the pool layout: a node's child block is followed by the regions of its
//      interior children in order (depth-first, the first child's block right behind its parent's);
//   4. every wide node's record, inline primitives and block padding are written in parallel (disjoint
//      ranges; the pool is never zero-filled).
// The tree depends only on the input (the splits are deterministic), so the pool is identical for any
// thread count and run.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <atomic>
#include <cmath>
#include <condition_variable>
#include <cstring>
#include <deque>
#include <limits>
#include <mutex>
#include <thread>

#include "pt_internal.h"

namespace pt {

namespace {

constexpr float kInf = std::numeric_limits<float>::infinity();

struct Box {
    float lo[3], hi[3];
    void empty() {
        for (int a = 0; a < 3; ++a) { lo[a] = kInf; hi[a] = -kInf; }
    }
    void grow(const Box& b) {
        for (int a = 0; a < 3; ++a) { lo[a] = std::min(lo[a], b.lo[a]); hi[a] = std::max(hi[a], b.hi[a]); }
    }
    void grow_pt(const float* p) {
        for (int a = 0; a < 3; ++a) { lo[a] = std::min(lo[a], p[a]); hi[a] = std::max(hi[a], p[a]); }
    }
    double area() const {
        double dx = (double)hi[0] - lo[0], dy = (double)hi[1] - lo[1], dz = (double)hi[2] - lo[2];
        if (dx < 0) return 0.0;
        return 2.0 * (dx * dy + dy * dz + dz * dx);
    }
};

// primitive reference: its exact fp32 box and id (32 B); the centroid is 0.5 (lo + hi)
struct Ref {
    Box b;
    uint32_t id;
    uint32_t pad;
    void centroid(float* c) const {
        for (int a = 0; a < 3; ++a) c[a] = 0.5f * (b.lo[a] + b.hi[a]);
    }
};
static_assert(sizeof(Ref) == 32, "Ref layout");


int n_workers(int64_t n) {
    unsigned hc = std::thread::hardware_concurrency();
    if (const char* e = std::getenv("PT_BVH_THREADS")) hc = (unsigned)std::max(1, std::atoi(e));
    if (hc == 0) hc = 1;
    if (n < 20000) return 1;
    return (int)std::min<unsigned>(hc, 64);
}

// ---- 1.+2. binned-SAH splits, collapsed to 4-wide nodes on the fly --------------------------------
// A wide node is built from its binary node: split it, then repeatedly split the largest-area interior
// child (the first one on equal areas) until it has 4 children or only leaves are left -- exactly the
// collapse of the full binary tree, without storing it. Every child's own split is decided here too
// (its leaf/interior kind and size go into the parent's record); an interior child carries its two
// binary children into its own task.
struct Item {
    int64_t first, count;
    Box bb, cb;   // bounds of the primitives and of their centroids
};

struct WChild {
    Box b;
    int32_t ref;     // leaf: first reference; interior: wide-node id
    int32_t count;   // leaf: primitive count; interior: 0
};
static_assert(sizeof(WChild) == 32, "WChild layout");

struct Wide {
    WChild c[4];
    int32_t nch = 0;
    int32_t depth = 1;
    int64_t block = 0;    // units of the child block (multiple of 4)
    int64_t region = 0;   // units of the child block plus the regions of all interior children
    int64_t rec = 0;      // unit of this node's 64-B record
    int64_t base = 0;     // unit of its child block
};

struct WideTask {
    int32_t id, depth;
    Item it, l, r;   // the node and its (already decided) binary split
};

struct Builder {
    // reference array and the partition scratch: uninitialised allocations (no serial zero fill of up to
    // 2 x 160 MB); the parallel fill and the chunked partition touch them first
    std::unique_ptr<Ref[]> refs_buf, scratch_buf;
    Ref* refs = nullptr;
    Ref* scratch = nullptr;
    int64_t n_refs = 0;
    std::vector<Wide> wide;          // preallocated (at most one wide node per primitive)
    std::atomic<int32_t> next_wide{1};
    std::atomic<int64_t> n_leaves{0};
    std::atomic<int32_t> max_depth{1};
    std::mutex mu;
    std::condition_variable cv;
    std::deque<WideTask> queue;
    int busy = 0;
    bool done = false;
    static constexpr int64_t kGrain = 2048;   // subtrees larger than this may move to another worker
    // nodes of at least kBigNode references (the top levels of large scenes, where few workers are busy)
    // are binned and partitioned by `helpers` threads over kChunks fixed chunks (fixed, so the result does
    // not depend on the thread count); `scratch` is the partition's buffer
    static constexpr int64_t kBigNode = 1 << 18;
    static constexpr int kChunks = 64;
    int helpers = 1;
    template <typename F>
    void chunked(int64_t n, F f) {
        std::atomic<int> next{0};
        auto run = [&] {
            for (int ch; (ch = next.fetch_add(1)) < kChunks;) f(ch, n * ch / kChunks, n * (ch + 1) / kChunks);
        };
        std::vector<std::thread> ts;
        for (int t = 1; t < helpers; ++t) ts.emplace_back(run);
        run();
        for (auto& t : ts) t.join();
    }
    static constexpr int NB = 32;   // max bins (nb <= NB used)
    // measured on configs 2-4 (profiles/round2/bvhparams_*.log): 32 bins, node cost 1.0 and leaves of at
    // most 2 primitives beat round 1's 16 / 1.5 / 4 by 1-3.5 % samples/s
    int nb = 32;                    // SAH bins (PT_BVH_BINS)
    double trav_cost = 1.0;         // node-traversal cost in primitive tests (PT_BVH_NODE_COST)
    int max_leaf = 2;               // leaf size cap (PT_BVH_MAX_LEAF, <= kMaxLeafPrims)

    void build(int threads) {
        const int64_t n = n_refs;
        wide.resize((size_t)std::max<int64_t>(1, n));
        Item root{0, n, {}, {}};
        root.bb.empty();
        root.cb.empty();
        for (int64_t i = 0; i < n; ++i) {
            const Ref& r = refs[i];
            float c[3];
            r.centroid(c);
            root.bb.grow(r.b);
            root.cb.grow_pt(c);
        }
        WideTask t0{0, 1, root, {}, {}};
        if (!split(root, t0.l, t0.r)) {     // one leaf: a root node with a single leaf child
            Wide& w = wide[0];
            w.nch = 1;
            w.c[0] = WChild{root.bb, 0, (int32_t)n};
            n_leaves = 1;
            next_wide = 1;
            return;
        }
        if (threads <= 1) {
            run_local(t0, false);
            return;
        }
        queue.push_back(t0);
        std::vector<std::thread> ws;
        for (int t = 0; t < threads; ++t) ws.emplace_back([this] { worker(); });
        for (auto& w : ws) w.join();
    }

    void worker() {
        for (;;) {
            WideTask t;
            {
                std::unique_lock<std::mutex> lk(mu);
                cv.wait(lk, [&] { return done || !queue.empty(); });
                if (queue.empty()) return;   // done
                t = queue.front();
                queue.pop_front();
                ++busy;
            }
            run_local(t, true);
            {
                std::lock_guard<std::mutex> lk(mu);
                --busy;
                if (busy == 0 && queue.empty()) {
                    done = true;
                    cv.notify_all();
                }
            }
        }
    }

    void run_local(const WideTask& top, bool share) {
        std::vector<WideTask> stack;
        stack.push_back(top);
        WideTask kids[4];
        while (!stack.empty()) {
            const WideTask t = stack.back();
            stack.pop_back();
            const int nk = make_wide(t, kids);
            for (int k = nk - 1; k >= 0; --k) {
                if (share && k > 0 && kids[k].it.count > kGrain) {
                    std::lock_guard<std::mutex> lk(mu);
                    if (queue.size() < 1024) {
                        queue.push_back(kids[k]);
                        cv.notify_one();
                        continue;
                    }
                }
                stack.push_back(kids[k]);
            }
        }
    }

    // Build wide node t.id from its split; returns its interior children's tasks.
    int make_wide(const WideTask& t, WideTask* kids) {
        struct Cand {
            Item it, l, r;
            int state;   // 0 undecided, 1 leaf, 2 interior (l, r valid)
        };
        Cand c[4];
        int nc = 2;
        c[0] = Cand{t.l, {}, {}, 0};
        c[1] = Cand{t.r, {}, {}, 0};
        auto decide = [&](Cand& x) {
            if (x.state == 0) x.state = split(x.it, x.l, x.r) ? 2 : 1;
        };
        while (nc < 4) {
            // the largest-area interior candidate (first on ties), deciding candidates as needed
            int best = -1;
            double ba = -1.0;
            bool retry = true;
            while (retry) {
                retry = false;
                best = -1;
                ba = -1.0;
                for (int i = 0; i < nc; ++i) {
                    if (c[i].state == 1) continue;
                    const double a = c[i].it.bb.area();
                    if (a > ba) { ba = a; best = i; }
                }
                if (best >= 0 && c[best].state == 0) {
                    decide(c[best]);
                    if (c[best].state == 1) retry = true;
                }
            }
            if (best < 0) break;
            const Cand e = c[best];
            for (int i = best; i + 1 < nc; ++i) c[i] = c[i + 1];
            --nc;
            c[nc++] = Cand{e.l, {}, {}, 0};
            c[nc++] = Cand{e.r, {}, {}, 0};
        }
        for (int i = 0; i < nc; ++i) decide(c[i]);
        Wide& w = wide[t.id];
        w.depth = t.depth;
        int nk = 0, o = 0;
        for (int pass = 0; pass < 2; ++pass) {          // interior children first, then leaves
            for (int i = 0; i < nc; ++i) {
                const bool interior = c[i].state == 2;
                if (interior != (pass == 0)) continue;
                if (interior) {
                    const int32_t id = next_wide.fetch_add(1);
                    w.c[o++] = WChild{c[i].it.bb, id, 0};
                    kids[nk++] = WideTask{id, t.depth + 1, c[i].it, c[i].l, c[i].r};
                } else {
                    w.c[o++] = WChild{c[i].it.bb, (int32_t)c[i].it.first, (int32_t)c[i].it.count};
                    n_leaves.fetch_add(1, std::memory_order_relaxed);
                }
            }
        }
        w.nch = o;
        int32_t md = max_depth.load(std::memory_order_relaxed);
        while (t.depth > md && !max_depth.compare_exchange_weak(md, t.depth)) {
        }
        return nk;
    }

    // Split one node (binned SAH over the widest centroid axis, node-traversal cost 1.5 primitive tests
    // per unit area), or decide it is a leaf. Returns true and the two children if it was split; the
    // references of the node are partitioned in place.
    bool split(const Item& it, Item& L, Item& R) {
        int axis = 0;
        float ext = it.cb.hi[0] - it.cb.lo[0];
        for (int a = 1; a < 3; ++a)
            if (it.cb.hi[a] - it.cb.lo[a] > ext) { ext = it.cb.hi[a] - it.cb.lo[a]; axis = a; }
        Ref* const r0 = refs + it.first;
        const int64_t cnt_all = it.count;
        int64_t split = -1;
        Box lb, lcb, rb, rcb;
        if (cnt_all > 1 && ext > 0.0f) {
            int64_t cnt[NB] = {0};
            Box bins[NB], cbins[NB];
            for (int k = 0; k < nb; ++k) { bins[k].empty(); cbins[k].empty(); }
            const float scale = (float)(nb / (double)ext);
            const float c0 = it.cb.lo[axis];
            auto bin_of = [&](const Ref& r) {
                const float c = 0.5f * (r.b.lo[axis] + r.b.hi[axis]);
                const int k = (int)((c - c0) * scale);
                return std::min(nb - 1, std::max(0, k));
            };
            const bool big = cnt_all >= kBigNode;   // (for any thread count: the same partition order)
            if (big) {
                // the top splits: bin fixed chunks on helper threads, reduce in chunk order (exactly the
                // serial bins: counts add, boxes unite)
                std::vector<int64_t> ccnt((size_t)kChunks * NB, 0);
                std::vector<Box> cb((size_t)kChunks * NB), ccb((size_t)kChunks * NB);
                for (auto& b : cb) b.empty();
                for (auto& b : ccb) b.empty();
                chunked(cnt_all, [&](int ch, int64_t b0, int64_t b1) {
                    for (int64_t i = b0; i < b1; ++i) {
                        const Ref& r = r0[i];
                        const int k = bin_of(r);
                        ccnt[(size_t)ch * NB + k]++;
                        cb[(size_t)ch * NB + k].grow(r.b);
                        float c[3];
                        r.centroid(c);
                        ccb[(size_t)ch * NB + k].grow_pt(c);
                    }
                });
                for (int ch = 0; ch < kChunks; ++ch)
                    for (int k = 0; k < nb; ++k) {
                        cnt[k] += ccnt[(size_t)ch * NB + k];
                        bins[k].grow(cb[(size_t)ch * NB + k]);
                        cbins[k].grow(ccb[(size_t)ch * NB + k]);
                    }
            } else {
                for (int64_t i = 0; i < cnt_all; ++i) {
                    const Ref& r = r0[i];
                    const int k = bin_of(r);
                    cnt[k]++;
                    bins[k].grow(r.b);
                    float c[3];
                    r.centroid(c);
                    cbins[k].grow_pt(c);
                }
            }
            double rarea[NB];
            int64_t rcnt[NB];
            Box acc;
            acc.empty();
            int64_t c = 0;
            for (int k = nb - 1; k >= 1; --k) {
                acc.grow(bins[k]);
                c += cnt[k];
                rarea[k] = acc.area();
                rcnt[k] = c;
            }
            double best = std::numeric_limits<double>::infinity();
            int best_k = -1;
            acc.empty();
            c = 0;
            for (int k = 0; k < nb - 1; ++k) {
                acc.grow(bins[k]);
                c += cnt[k];
                if (c == 0 || rcnt[k + 1] == 0) continue;
                const double cost = acc.area() * (double)c + rarea[k + 1] * (double)rcnt[k + 1];
                if (cost < best) { best = cost; best_k = k; }
            }
            const double kTraversalCost = trav_cost;
            const double leaf_cost = it.bb.area() * (double)cnt_all;
            best += kTraversalCost * it.bb.area();
            if (best_k >= 0 && (best < leaf_cost || cnt_all > max_leaf)) {
                if (big) {
                    // stable partition in fixed chunks: count, prefix, scatter into the scratch, copy back
                    std::vector<int64_t> nl(kChunks, 0);
                    chunked(cnt_all, [&](int ch, int64_t b0, int64_t b1) {
                        int64_t m = 0;
                        for (int64_t i = b0; i < b1; ++i) m += bin_of(r0[i]) <= best_k;
                        nl[ch] = m;
                    });
                    int64_t left = 0;
                    for (int ch = 0; ch < kChunks; ++ch) left += nl[ch];
                    std::vector<int64_t> lo_at(kChunks), hi_at(kChunks);
                    int64_t a = 0, b = left;
                    for (int ch = 0; ch < kChunks; ++ch) {
                        const int64_t b0 = cnt_all * ch / kChunks, b1 = cnt_all * (ch + 1) / kChunks;
                        lo_at[ch] = a;
                        hi_at[ch] = b;
                        a += nl[ch];
                        b += (b1 - b0) - nl[ch];
                    }
                    Ref* tmp = scratch + it.first;
                    chunked(cnt_all, [&](int ch, int64_t b0, int64_t b1) {
                        int64_t pl = lo_at[ch], ph = hi_at[ch];
                        for (int64_t i = b0; i < b1; ++i) tmp[bin_of(r0[i]) <= best_k ? pl++ : ph++] = r0[i];
                    });
                    chunked(cnt_all, [&](int, int64_t b0, int64_t b1) {
                        std::memcpy(r0 + b0, tmp + b0, sizeof(Ref) * (size_t)(b1 - b0));
                    });
                    split = it.first + left;
                } else {
                    Ref* mid = std::partition(r0, r0 + cnt_all, [&](const Ref& r) { return bin_of(r) <= best_k; });
                    split = it.first + (mid - r0);
                }
                lb.empty(); lcb.empty(); rb.empty(); rcb.empty();
                for (int k = 0; k < nb; ++k) {
                    if (k <= best_k) { lb.grow(bins[k]); lcb.grow(cbins[k]); }
                    else { rb.grow(bins[k]); rcb.grow(cbins[k]); }
                }
            }
        } else if (cnt_all > max_leaf) {
            split = it.first + cnt_all / 2;   // coincident centroids
            lb.empty(); lcb.empty(); rb.empty(); rcb.empty();
            for (int64_t i = 0; i < cnt_all; ++i) {
                float c[3];
                r0[i].centroid(c);
                if (it.first + i < split) { lb.grow(r0[i].b); lcb.grow_pt(c); }
                else { rb.grow(r0[i].b); rcb.grow_pt(c); }
            }
        }
        if (split > it.first && split < it.first + cnt_all) {
            L = Item{it.first, split - it.first, lb, lcb};
            R = Item{split, it.first + cnt_all - split, rb, rcb};
            return true;
        }
        return false;
    }
};

inline float f32_next_down(double x) {
    float f = (float)x;
    if ((double)f > x) f = std::nextafter(f, -kInf);
    return f;
}
inline float f32_next_up(double x) {
    float f = (float)x;
    if ((double)f < x) f = std::nextafter(f, kInf);
    return f;
}

// The node origin with 4 metadata bits embedded in its lowest mantissa bits: a float <= lo (so every
// child offset stays >= 0) whose low 4 bits are `nib` -- 16 ulps below lo, then the bits replaced
// (positive: the value rises by at most 15 ulps; negative: the magnitude falls by at most 15 ulps).
inline float embed_nibble(float lo, uint32_t nib) {
    float x = lo;
    for (int i = 0; i < 16; ++i) x = std::nextafter(x, -kInf);
    uint32_t b = __builtin_bit_cast(uint32_t, x);
    b = (b & ~15u) | (nib & 15u);
    return __builtin_bit_cast(float, b);
}

inline float decode(float O, uint16_t h) {
    volatile float hv = (float)f16_value(h);   // exact widening
    volatile float s = O + hv;                 // the single fp32 round-to-nearest add the kernel does
    return s;
}

template <typename F>
void parallel_for(int threads, int64_t n, F f) {
    if (threads <= 1 || n < 1024) {
        for (int64_t i = 0; i < n; ++i) f(i);
        return;
    }
    std::atomic<int64_t> next{0};
    constexpr int64_t kChunk = 512;
    std::vector<std::thread> ws;
    for (int t = 0; t < threads; ++t)
        ws.emplace_back([&] {
            for (;;) {
                const int64_t s = next.fetch_add(kChunk);
                if (s >= n) return;
                const int64_t e = std::min(n, s + kChunk);
                for (int64_t i = s; i < e; ++i) f(i);
            }
        });
    for (auto& w : ws) w.join();
}

}  // namespace

double f16_value(uint16_t h) {
    int e = (h >> 10) & 31, m = h & 1023;
    double v;
    if (e == 0) v = std::ldexp((double)m, -24);
    else if (e == 31) v = m ? std::numeric_limits<double>::quiet_NaN() : std::numeric_limits<double>::infinity();
    else v = std::ldexp((double)(m | 1024), e - 25);
    return (h & 0x8000) ? -v : v;
}

// Largest binary16 <= x, for 0 <= x <= 65504.
uint16_t f16_round_down(double x) {
    if (!(x > 0.0)) return 0;
    if (x >= 65504.0) return 0x7BFF;
    int e;
    std::frexp(x, &e);          // x = f * 2^e, f in [0.5, 1)
    int ex = e - 1;             // x in [2^ex, 2^(ex+1))
    if (ex < -14) {             // subnormal range: step 2^-24
        double m = std::floor(std::ldexp(x, 24));
        return (uint16_t)m;
    }
    double m = std::floor(std::ldexp(x, 10 - ex));   // in [1024, 2047]
    return (uint16_t)(((ex + 15) << 10) | ((int)m - 1024));
}

// Smallest binary16 >= x ("round-to-nearest-not-lower" SPEC.md:36-44 generalised), 0 <= x <= 65504.
uint16_t f16_round_up(double x) {
    uint16_t h = f16_round_down(x);
    if (f16_value(h) < x) ++h;   // positive halves are ordered like their bit patterns
    return h;
}

int build_wide_bvh(const pt_triangle* tris, int64_t n_tris, const pt_sphere* sph, int64_t n_sph, HostBvh* out,
                   std::string* msg) {
    const int64_t n = n_tris + n_sph;
    out->pool.reset();
    out->units = 0;
    out->empty = (n == 0);
    out->n_nodes = out->n_leaves = out->max_depth = 0;
    if (n == 0) return PT_OK;
    const int threads = n_workers(n);
    static const bool timing = std::getenv("PT_BVH_TIMING") != nullptr;
    auto now = [] { return std::chrono::steady_clock::now(); };
    auto t0 = now();
    auto lap = [&](const char* what) {
        if (!timing) return;
        auto t1 = now();
        std::fprintf(stderr, "bvh %-10s %8.2f ms (%d threads)\n", what,
                     std::chrono::duration<double, std::milli>(t1 - t0).count(), threads);
        t0 = t1;
    };
    if (n >= (1ll << 30)) { *msg = "too many primitives for the BVH builder (< 2^30)"; return PT_ERR_INVALID_ARG; }
    Builder B;
    // tuning knobs (experiments; defaults = the measured configuration)
    if (const char* e = std::getenv("PT_BVH_BINS")) B.nb = std::max(2, std::min(Builder::NB, std::atoi(e)));
    if (const char* e = std::getenv("PT_BVH_NODE_COST")) B.trav_cost = std::atof(e);
    if (const char* e = std::getenv("PT_BVH_MAX_LEAF")) B.max_leaf = std::max(1, std::min(kMaxLeafPrims, std::atoi(e)));
    B.refs_buf.reset(new Ref[(size_t)n]);
    B.refs = B.refs_buf.get();
    B.n_refs = n;
    B.helpers = threads;
    if (n >= Builder::kBigNode) {
        B.scratch_buf.reset(new Ref[(size_t)n]);
        B.scratch = B.scratch_buf.get();
    }
    parallel_for(threads, n, [&](int64_t i) {
        Ref& r = B.refs[i];
        r.id = (uint32_t)i;
        r.pad = 0;
        if (i < n_tris) {
            const pt_triangle& t = tris[i];
            for (int a = 0; a < 3; ++a) {
                r.b.lo[a] = std::min(t.v0[a], std::min(t.v1[a], t.v2[a]));
                r.b.hi[a] = std::max(t.v0[a], std::max(t.v1[a], t.v2[a]));
            }
        } else {
            const pt_sphere& s = sph[i - n_tris];
            for (int a = 0; a < 3; ++a) {
                r.b.lo[a] = f32_next_down((double)s.center[a] - (double)s.radius);
                r.b.hi[a] = f32_next_up((double)s.center[a] + (double)s.radius);
            }
        }
    });
    lap("refs");
    B.build(threads);
    lap("wide");
    const int64_t n_wide = B.next_wide.load();
    std::vector<Wide>& W = B.wide;
    // ---- 3. layout: block sizes, regions (children have larger ids than parents: reverse order), then
    // bases in id order (a node's base depends only on its parent's base and its earlier siblings) ----
    for (int64_t wi = n_wide - 1; wi >= 0; --wi) {
        Wide& w = W[wi];
        int64_t units = 0, region = 0;
        for (int i = 0; i < w.nch; ++i) {
            if (w.c[i].count == 0) {
                units += kNodeUnits;
                region += W[w.c[i].ref].region;
            } else {
                units += (int64_t)kPrimUnits * w.c[i].count;
            }
        }
        w.block = (units + 3) & ~int64_t(3);
        w.region = w.block + region;
    }
    const int64_t total = (int64_t)kNodeUnits + W[0].region;
    if (total > (1ll << 28)) { *msg = "BVH pool exceeds 2^28 units (4 GiB)"; return PT_ERR_DOMAIN; }
    W[0].rec = 0;
    W[0].base = kNodeUnits;
    for (int64_t wi = 0; wi < n_wide; ++wi) {
        const Wide& w = W[wi];
        int64_t next = w.base + w.block;
        for (int i = 0; i < w.nch; ++i) {
            if (w.c[i].count != 0) continue;
            Wide& c = W[w.c[i].ref];
            c.rec = w.base + (int64_t)kNodeUnits * i;   // interior children lead the block
            c.base = next;
            next += c.region;
        }
    }
    lap("layout");
    // every unit is written below (records, inline primitives, block padding): no zero fill
    out->pool.reset(new uint4[(size_t)total]);
    out->units = total;
    uint4* pool = out->pool.get();
    const Ref* refs = B.refs;
    lap("alloc");

    // ---- 4. records and inline primitives, in parallel ----
    std::atomic<int> err{0};
    std::mutex err_mu;
    parallel_for(threads, n_wide, [&](int64_t wi) {
        const Wide& w = W[wi];
        // Child metadata: one nibble per child = its size in pool units (0: no child, 4: interior node,
        // 3 * count: leaf of count primitives), so the kernel gets validity, kind, count and the running
        // child offset from one 16-bit field: nibbles 0-2 ride in the low mantissa bits of the origin's
        // x, y, z (embed_nibble), nibble 3 in the top bits of the base.
        uint32_t nib[4] = {0, 0, 0, 0};
        Box nb;
        nb.empty();
        for (int ci = 0; ci < w.nch; ++ci) {
            const WChild& c = w.c[ci];
            nib[ci] = c.count > 0 ? (uint32_t)(kPrimUnits * c.count) : (uint32_t)kNodeUnits;
            nb.grow(c.b);
        }
        float Oq[3];
        for (int a = 0; a < 3; ++a) Oq[a] = embed_nibble(nb.lo[a], nib[a]);
        uint4& h0 = pool[w.rec];
        h0.x = __builtin_bit_cast(uint32_t, Oq[0]);
        h0.y = __builtin_bit_cast(uint32_t, Oq[1]);
        h0.z = __builtin_bit_cast(uint32_t, Oq[2]);
        h0.w = (uint32_t)w.base | (nib[3] << 28);
        uint16_t q[4][6];
        std::memset(q, 0, sizeof(q));
        int64_t off = w.base;
        for (int ci = 0; ci < w.nch; ++ci) {
            const WChild& c = w.c[ci];
            for (int a = 0; a < 3; ++a) {
                const float O = Oq[a];
                const double dlo = (double)c.b.lo[a] - (double)O, dhi = (double)c.b.hi[a] - (double)O;
                if (!(dhi <= 65504.0) || !(dlo >= 0.0)) {
                    std::lock_guard<std::mutex> lk(err_mu);
                    if (!err.exchange(1))
                        *msg = "child box offset outside the fp16 range (scene extent too large for one node)";
                    return;
                }
                uint16_t hl = f16_round_down(dlo);
                while (hl > 0 && decode(O, hl) > c.b.lo[a]) --hl;
                uint16_t hh = f16_round_up(dhi);
                while (decode(O, hh) < c.b.hi[a]) {
                    if (hh >= 0x7BFF) {
                        std::lock_guard<std::mutex> lk(err_mu);
                        if (!err.exchange(1)) *msg = "child box hi beyond fp16 range";
                        return;
                    }
                    ++hh;
                }
                q[ci][a] = hl;
                q[ci][3 + a] = hh;
            }
            if (c.count > 0) {
                for (int64_t k = 0; k < c.count; ++k) {
                    const uint32_t id = refs[c.ref + k].id;
                    uint4* u = &pool[off + kPrimUnits * k];
                    // material bits ride in the spare words, so shading reads the hit primitive from here
                    if ((int64_t)id < n_tris) {
                        const pt_triangle& t = tris[id];
                        u[0] = make_uint4(__builtin_bit_cast(uint32_t, t.v0[0]), __builtin_bit_cast(uint32_t, t.v0[1]),
                                          __builtin_bit_cast(uint32_t, t.v0[2]), id);
                        u[1] = make_uint4(__builtin_bit_cast(uint32_t, t.v1[0]), __builtin_bit_cast(uint32_t, t.v1[1]),
                                          __builtin_bit_cast(uint32_t, t.v1[2]), t.material);
                        u[2] = make_uint4(__builtin_bit_cast(uint32_t, t.v2[0]), __builtin_bit_cast(uint32_t, t.v2[1]),
                                          __builtin_bit_cast(uint32_t, t.v2[2]), 0u);
                    } else {
                        const pt_sphere& s = sph[id - n_tris];
                        u[0] = make_uint4(__builtin_bit_cast(uint32_t, s.center[0]),
                                          __builtin_bit_cast(uint32_t, s.center[1]),
                                          __builtin_bit_cast(uint32_t, s.center[2]), id | kSphereFlag);
                        u[1] = make_uint4(__builtin_bit_cast(uint32_t, s.radius), s.material, 0u, 0u);
                        u[2] = make_uint4(0u, 0u, 0u, 0u);
                    }
                }
                off += (int64_t)kPrimUnits * c.count;
            } else {
                off += kNodeUnits;
            }
        }
        for (int64_t u = off; u < w.base + w.block; ++u) pool[u] = make_uint4(0, 0, 0, 0);   // block padding
        // pack the 4 x 12-B child records into units 1..3: one word per axis, (lo | hi << 16), so the
        // kernel decodes both bounds of an axis with one packed fp16x2 -> fp32x2 conversion
        uint32_t words[12];
        for (int ci = 0; ci < 4; ++ci)
            for (int a = 0; a < 3; ++a) words[3 * ci + a] = (uint32_t)q[ci][a] | ((uint32_t)q[ci][3 + a] << 16);
        pool[w.rec + 1] = make_uint4(words[0], words[1], words[2], words[3]);
        pool[w.rec + 2] = make_uint4(words[4], words[5], words[6], words[7]);
        pool[w.rec + 3] = make_uint4(words[8], words[9], words[10], words[11]);
    });
    lap("fill");
    if (err.load()) {
        out->pool.reset();
        out->units = 0;
        return PT_ERR_DOMAIN;
    }
    out->n_nodes = n_wide;
    out->n_leaves = B.n_leaves.load();
    out->max_depth = B.max_depth.load();
    const int64_t maxd = out->max_depth;
    if (3 * maxd + 4 > kStackSize) { *msg = "BVH too deep for the traversal stack"; return PT_ERR_DOMAIN; }
    return PT_OK;
}

}  // namespace pt
