// bvh_build.cpp -- host builder of the 4-wide compressed BVH (Sec. 3.1.4).
//
// The paper builds a BVH-2 on the host (Embree), compacts it into pointer-less nodes whose first
// child is implicit, and stores box extents in fp16 with "round-to-nearest-not-lower" so no
// intersection can be missed. Here: a binned-SAH BVH-2 (16 bins, leaves <= 4 primitives) is collapsed
// into 4-wide nodes (largest-area interior child expanded first), children are stored contiguously
// behind one base index, leaf primitives are stored inline, and each child box is quantised to fp16
// offsets from the node origin -- lo rounded down, hi rounded up, then corrected until the exact fp32
// decode the traversal kernel performs (O + f16) contains the exact box. Every node is re-verified.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <limits>

#include "pt_internal.h"

namespace pt {

namespace {

struct Box {
    float lo[3], hi[3];
    void empty() {
        for (int a = 0; a < 3; ++a) { lo[a] = std::numeric_limits<float>::infinity(); hi[a] = -lo[a]; }
    }
    void grow(const Box& b) {
        for (int a = 0; a < 3; ++a) { lo[a] = std::min(lo[a], b.lo[a]); hi[a] = std::max(hi[a], b.hi[a]); }
    }
    double area() const {
        double dx = (double)hi[0] - lo[0], dy = (double)hi[1] - lo[1], dz = (double)hi[2] - lo[2];
        if (dx < 0) return 0.0;
        return 2.0 * (dx * dy + dy * dz + dz * dx);
    }
};

struct Node2 {
    Box b;
    int32_t left = -1, right = -1;
    int32_t first = 0, count = 0;  // leaf iff count > 0
};

struct Builder {
    std::vector<Box> pbox;
    std::vector<float> cen;  // [n][3]
    std::vector<int64_t> order;
    std::vector<Node2> nodes;

    void build(int64_t n) {
        order.resize(n);
        for (int64_t i = 0; i < n; ++i) order[i] = i;
        nodes.reserve(2 * n + 1);
        nodes.emplace_back();
        struct Item { int64_t node, first, count; };
        std::vector<Item> stack;
        stack.push_back({0, 0, n});
        constexpr int NB = 16;
        while (!stack.empty()) {
            Item it = stack.back();
            stack.pop_back();
            Box bb, cb;
            bb.empty();
            cb.empty();
            for (int64_t i = it.first; i < it.first + it.count; ++i) {
                int64_t id = order[i];
                bb.grow(pbox[id]);
                for (int a = 0; a < 3; ++a) {
                    cb.lo[a] = std::min(cb.lo[a], cen[3 * id + a]);
                    cb.hi[a] = std::max(cb.hi[a], cen[3 * id + a]);
                }
            }
            nodes[it.node].b = bb;
            int axis = 0;
            float ext = cb.hi[0] - cb.lo[0];
            for (int a = 1; a < 3; ++a)
                if (cb.hi[a] - cb.lo[a] > ext) { ext = cb.hi[a] - cb.lo[a]; axis = a; }
            int64_t split = -1;
            if (it.count > 1 && ext > 0.0f) {
                int64_t cnt[NB] = {0};
                Box bins[NB];
                for (auto& b : bins) b.empty();
                const double scale = NB / (double)ext;
                auto bin_of = [&](int64_t id) {
                    int k = (int)(((double)cen[3 * id + axis] - cb.lo[axis]) * scale);
                    return std::min(NB - 1, std::max(0, k));
                };
                for (int64_t i = it.first; i < it.first + it.count; ++i) {
                    int64_t id = order[i];
                    int k = bin_of(id);
                    cnt[k]++;
                    bins[k].grow(pbox[id]);
                }
                // prefix/suffix sweeps
                double rarea[NB];
                int64_t rcnt[NB];
                Box acc;
                acc.empty();
                int64_t c = 0;
                for (int k = NB - 1; k >= 1; --k) {
                    acc.grow(bins[k]);
                    c += cnt[k];
                    rarea[k] = acc.area();
                    rcnt[k] = c;
                }
                double best = std::numeric_limits<double>::infinity();
                int best_k = -1;
                acc.empty();
                c = 0;
                for (int k = 0; k < NB - 1; ++k) {
                    acc.grow(bins[k]);
                    c += cnt[k];
                    if (c == 0 || rcnt[k + 1] == 0) continue;
                    double cost = acc.area() * (double)c + rarea[k + 1] * (double)rcnt[k + 1];
                    if (cost < best) { best = cost; best_k = k; }
                }
                // SAH with a node-traversal cost of kTraversalCost primitive tests (per unit area)
                constexpr double kTraversalCost = 1.5;
                double leaf_cost = bb.area() * (double)it.count;
                best += kTraversalCost * bb.area();
                if (best_k >= 0 && (best < leaf_cost || it.count > kMaxLeafPrims)) {
                    auto mid = std::partition(order.begin() + it.first, order.begin() + it.first + it.count,
                                              [&](int64_t id) { return bin_of(id) <= best_k; });
                    split = mid - order.begin();
                }
            } else if (it.count > kMaxLeafPrims) {
                split = it.first + it.count / 2;  // coincident centroids
            }
            if (split > it.first && split < it.first + it.count) {
                int64_t l = (int64_t)nodes.size();
                nodes.emplace_back();
                nodes.emplace_back();
                nodes[it.node].left = (int32_t)l;
                nodes[it.node].right = (int32_t)(l + 1);
                stack.push_back({l + 1, split, it.first + it.count - split});
                stack.push_back({l, it.first, split - it.first});
            } else {
                nodes[it.node].first = (int32_t)it.first;
                nodes[it.node].count = (int32_t)it.count;
            }
        }
    }
};

inline float f32_next_down(double x) {
    float f = (float)x;
    if ((double)f > x) f = std::nextafter(f, -std::numeric_limits<float>::infinity());
    return f;
}
inline float f32_next_up(double x) {
    float f = (float)x;
    if ((double)f < x) f = std::nextafter(f, std::numeric_limits<float>::infinity());
    return f;
}

// The node origin with 4 metadata bits embedded in its lowest mantissa bits: a float <= lo (so every
// child offset stays >= 0) whose low 4 bits are `nib` -- 16 ulps below lo, then the bits replaced
// (positive: the value rises by at most 15 ulps; negative: the magnitude falls by at most 15 ulps).
inline float embed_nibble(float lo, uint32_t nib) {
    float x = lo;
    for (int i = 0; i < 16; ++i) x = std::nextafter(x, -std::numeric_limits<float>::infinity());
    uint32_t b = __builtin_bit_cast(uint32_t, x);
    b = (b & ~15u) | (nib & 15u);
    return __builtin_bit_cast(float, b);
}

inline float decode(float O, uint16_t h) {
    volatile float hv = (float)f16_value(h);   // exact widening
    volatile float s = O + hv;                 // the single fp32 round-to-nearest add the kernel does
    return s;
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
    out->pool.clear();
    out->empty = (n == 0);
    out->n_nodes = out->n_leaves = out->max_depth = 0;
    if (n == 0) return PT_OK;
    Builder B;
    B.pbox.resize(n);
    B.cen.resize(3 * n);
    for (int64_t i = 0; i < n; ++i) {
        Box& b = B.pbox[i];
        if (i < n_tris) {
            const pt_triangle& t = tris[i];
            for (int a = 0; a < 3; ++a) {
                b.lo[a] = std::min(t.v0[a], std::min(t.v1[a], t.v2[a]));
                b.hi[a] = std::max(t.v0[a], std::max(t.v1[a], t.v2[a]));
            }
        } else {
            const pt_sphere& s = sph[i - n_tris];
            for (int a = 0; a < 3; ++a) {
                b.lo[a] = f32_next_down((double)s.center[a] - (double)s.radius);
                b.hi[a] = f32_next_up((double)s.center[a] + (double)s.radius);
            }
        }
        for (int a = 0; a < 3; ++a) B.cen[3 * i + a] = 0.5f * (b.lo[a] + b.hi[a]);
    }
    B.build(n);

    // ---- collapse to 4-wide + layout ----------------------------------------------------------
    std::vector<uint4>& pool = out->pool;
    auto alloc = [&](int64_t units) {
        int64_t at = (int64_t)pool.size();
        pool.resize(at + units, make_uint4(0, 0, 0, 0));
        return at;
    };
    struct Pending { int32_t n2; int64_t unit; int64_t depth; };
    std::vector<Pending> work;
    alloc(kNodeUnits);
    work.push_back({0, 0, 1});
    int64_t n_nodes = 0, n_leaves = 0, maxd = 0;
    while (!work.empty()) {
        Pending pnd = work.back();
        work.pop_back();
        ++n_nodes;
        maxd = std::max(maxd, pnd.depth);
        std::vector<int32_t> ch;
        const Node2& root2 = B.nodes[pnd.n2];
        if (root2.count > 0) ch.push_back(pnd.n2);   // whole scene is one leaf
        else { ch.push_back(root2.left); ch.push_back(root2.right); }
        while ((int)ch.size() < 4) {
            int best = -1;
            double ba = -1.0;
            for (int i = 0; i < (int)ch.size(); ++i) {
                const Node2& c = B.nodes[ch[i]];
                if (c.count == 0 && c.b.area() > ba) { ba = c.b.area(); best = i; }
            }
            if (best < 0) break;
            int32_t e = ch[best];
            ch.erase(ch.begin() + best);
            ch.push_back(B.nodes[e].left);
            ch.push_back(B.nodes[e].right);
        }
        // interior children first, then leaves
        std::stable_partition(ch.begin(), ch.end(), [&](int32_t c) { return B.nodes[c].count == 0; });
        int64_t units = 0;
        for (int32_t c : ch) units += B.nodes[c].count == 0 ? kNodeUnits : (int64_t)kPrimUnits * B.nodes[c].count;
        units = (units + 3) & ~int64_t(3);
        int64_t base = alloc(units);
        if (base + units > (1ll << 28)) { *msg = "BVH pool exceeds 2^28 units (4 GiB)"; return PT_ERR_DOMAIN; }
        // node header. Child metadata: one nibble per child = its size in pool units (0: no child,
        // 4: interior node, 3 * count: leaf of count primitives), so the kernel gets validity, kind,
        // count and the running child offset from one 16-bit field: nibbles 0-2 ride in the low
        // mantissa bits of the origin's x, y, z (embed_nibble), nibble 3 in the top bits of the base.
        uint32_t nib[4] = {0, 0, 0, 0};
        for (int ci = 0; ci < (int)ch.size(); ++ci) {
            const Node2& c = B.nodes[ch[ci]];
            nib[ci] = c.count > 0 ? (uint32_t)(kPrimUnits * c.count) : (uint32_t)kNodeUnits;
        }
        Box nb;
        nb.empty();
        for (int32_t c : ch) nb.grow(B.nodes[c].b);
        float Oq[3];
        for (int a = 0; a < 3; ++a) Oq[a] = embed_nibble(nb.lo[a], nib[a]);
        uint4& h0 = pool[pnd.unit];
        h0.x = __builtin_bit_cast(uint32_t, Oq[0]);
        h0.y = __builtin_bit_cast(uint32_t, Oq[1]);
        h0.z = __builtin_bit_cast(uint32_t, Oq[2]);
        h0.w = (uint32_t)base | (nib[3] << 28);
        uint16_t q[4][6];
        std::memset(q, 0, sizeof(q));
        int64_t off = base;
        for (int ci = 0; ci < (int)ch.size(); ++ci) {
            const Node2& c = B.nodes[ch[ci]];
            for (int a = 0; a < 3; ++a) {
                const float O = Oq[a];
                double dlo = (double)c.b.lo[a] - (double)O, dhi = (double)c.b.hi[a] - (double)O;
                if (!(dhi <= 65504.0) || !(dlo >= 0.0)) {
                    *msg = "child box offset outside the fp16 range (scene extent too large for one node)";
                    return PT_ERR_DOMAIN;
                }
                uint16_t hl = f16_round_down(dlo);
                while (hl > 0 && decode(O, hl) > c.b.lo[a]) --hl;
                uint16_t hh = f16_round_up(dhi);
                while (decode(O, hh) < c.b.hi[a]) {
                    if (hh >= 0x7BFF) { *msg = "child box hi beyond fp16 range"; return PT_ERR_DOMAIN; }
                    ++hh;
                }
                q[ci][a] = hl;
                q[ci][3 + a] = hh;
            }
            const bool leaf = c.count > 0;
            if (leaf) {
                ++n_leaves;
                for (int k = 0; k < c.count; ++k) {
                    int64_t id = B.order[c.first + k];
                    uint4* u = &pool[off + kPrimUnits * k];
                    if (id < n_tris) {
                        const pt_triangle& t = tris[id];
                        u[0] = make_uint4(__builtin_bit_cast(uint32_t, t.v0[0]), __builtin_bit_cast(uint32_t, t.v0[1]),
                                          __builtin_bit_cast(uint32_t, t.v0[2]), (uint32_t)id);
                        u[1] = make_uint4(__builtin_bit_cast(uint32_t, t.v1[0]), __builtin_bit_cast(uint32_t, t.v1[1]),
                                          __builtin_bit_cast(uint32_t, t.v1[2]), 0u);
                        u[2] = make_uint4(__builtin_bit_cast(uint32_t, t.v2[0]), __builtin_bit_cast(uint32_t, t.v2[1]),
                                          __builtin_bit_cast(uint32_t, t.v2[2]), 0u);
                    } else {
                        const pt_sphere& s = sph[id - n_tris];
                        u[0] = make_uint4(__builtin_bit_cast(uint32_t, s.center[0]),
                                          __builtin_bit_cast(uint32_t, s.center[1]),
                                          __builtin_bit_cast(uint32_t, s.center[2]), (uint32_t)id | kSphereFlag);
                        u[1] = make_uint4(__builtin_bit_cast(uint32_t, s.radius), 0u, 0u, 0u);
                        u[2] = make_uint4(0u, 0u, 0u, 0u);
                    }
                }
                off += (int64_t)kPrimUnits * c.count;
            } else {
                work.push_back({ch[ci], off, pnd.depth + 1});
                off += kNodeUnits;
            }
        }
        // pack the 4 x 12-B child records into units 1..3: one word per axis, (lo | hi << 16), so the
        // kernel decodes both bounds of an axis with one packed fp16x2 -> fp32x2 conversion
        uint32_t words[12];
        for (int ci = 0; ci < 4; ++ci)
            for (int a = 0; a < 3; ++a) words[3 * ci + a] = (uint32_t)q[ci][a] | ((uint32_t)q[ci][3 + a] << 16);
        pool[pnd.unit + 1] = make_uint4(words[0], words[1], words[2], words[3]);
        pool[pnd.unit + 2] = make_uint4(words[4], words[5], words[6], words[7]);
        pool[pnd.unit + 3] = make_uint4(words[8], words[9], words[10], words[11]);
    }
    out->n_nodes = n_nodes;
    out->n_leaves = n_leaves;
    out->max_depth = maxd;
    if (3 * maxd + 4 > kStackSize) { *msg = "BVH too deep for the traversal stack"; return PT_ERR_DOMAIN; }
    return PT_OK;
}

}  // namespace pt
