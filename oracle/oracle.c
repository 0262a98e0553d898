/*
 * oracle.c -- plain, slow, fp64 CPU path tracer: the parity ORACLE for the B200 hot path.
 *
 * TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference leg may load this library. It shares no code, header, table or constant
 * generator with the CUDA path (paper_2305_20061_b200/csrc); it reads the same seeded input
 * arrays (paper_2305_20061_b200/scenes.py), whose byte layout it declares independently below.
 *
 * What it computes (citations: PAPER.md = /root/reference/PAPER.md line, SURVEY = /root/repo/SURVEY.md
 * section; DESIGN.md "Readings" lists every reading taken where the paper is silent):
 *   - Monte Carlo path tracing with no light sampling, contributions only from emitters hit by chance
 *     or escaped rays times the environment (Sec. 3.1);
 *   - Russian roulette "with probability proportional to their radiometric throughput" from depth 3
 *     (PAPER.md:78, 150), q = min(1, max beta) (reading R8);
 *   - environment = HDR-NIF: equirect (u,v) of the escape direction -> MLP -> exp;
 *     the MLP is BASELINE.json's SIREN (reading R1/R2);
 *   - closest hit by brute-force definition, accelerated by a plain binned-SAH BVH-2 whose result
 *     equals brute force bit-for-bit (the BVH is the oracle's own, not the GPU's);
 *   - triangle test: watertight ray/triangle (Woop, Benthin, Wald 2013), which PBRT-v3 uses
 *     ("derived from PBRT-v3"), in fp64;
 *   - RNG: Philox-4x32-10 (Salmon et al., SC'11) keyed by (pixel, sample, bounce) per BASELINE.json
 *     north_star, replacing the IPU's hardware xoshiro generator.
 * Floating point: fp64 everywhere except camera-ray generation, which is specified in IEEE fp32
 * (reading R22, SURVEY 8c precision plan) and widened exactly. Compile with
 * -ffp-contract=off so no operation is fused.
 *
 * Parity pins: tests/test_oracle_*.py (brute force, closed forms, furnace cases, library routines).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define EXPORT __attribute__((visibility("default")))

/* ---------------------------------------------------------------------------------------------- */
/* Input byte layouts (declared independently of include/pt.h; the layout is the input format)      */
/* ---------------------------------------------------------------------------------------------- */
typedef struct { float v0[3], v1[3], v2[3]; uint32_t material; } in_tri;           /* 40 B */
typedef struct { float c[3]; float r; uint32_t material; } in_sphere;             /* 20 B */
typedef struct { uint32_t kind; float albedo[3]; float emission[3]; float ior; } in_mat; /* 32 B */
typedef struct { float eye[3], look_at[3], up[3]; float vfov_deg; } in_cam;       /* 40 B */

enum { K_LAMBERT = 0, K_MIRROR = 1, K_DIELECTRIC = 2, K_EMISSIVE = 3 };

/* ---------------------------------------------------------------------------------------------- */
/* Philox-4x32-10 (Salmon, Moraes, Dror, Shaw, "Parallel random numbers: as easy as 1, 2, 3", SC'11) */
/* ---------------------------------------------------------------------------------------------- */
static void philox4x32_10(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4]) {
    uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
    uint32_t k0 = key_in[0], k1 = key_in[1];
    for (int round = 0; round < 10; ++round) {
        uint64_t p0 = (uint64_t)0xD2511F53u * c0;
        uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
        uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
        uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
        uint32_t n0 = hi1 ^ c1 ^ k0;
        uint32_t n1 = lo1;
        uint32_t n2 = hi0 ^ c3 ^ k1;
        uint32_t n3 = lo0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* u = (x >> 8) * 2^-24 in [0, 1 - 2^-24]: exact in fp32 and fp64 (reading R13). */
static double u01(uint32_t x) { return (double)(x >> 8) * (1.0 / 16777216.0); }

/* Draw the 4 uniforms of (pixel p, sample s, slot) from stream 0, key = seed (R13). */
static void draw4(uint64_t seed, uint32_t p, uint32_t s, uint32_t slot, double u[4]) {
    uint32_t ctr[4] = {p, s, slot, 0u};
    uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
    uint32_t o[4];
    philox4x32_10(ctr, key, o);
    for (int i = 0; i < 4; ++i) u[i] = u01(o[i]);
}

EXPORT void orc_philox(const uint32_t* ctr, const uint32_t* key, int64_t n, uint32_t* out) {
    for (int64_t i = 0; i < n; ++i) philox4x32_10(ctr + 4 * i, key + 2 * i, out + 4 * i);
}

/* ---------------------------------------------------------------------------------------------- */
/* Scene + BVH-2 (binned SAH). The BVH only accelerates; closest_hit == brute force (tests pin it).   */
/* ---------------------------------------------------------------------------------------------- */
typedef struct { double lo[3], hi[3]; } box3;
typedef struct { box3 b; int32_t left, right; int32_t first, count; } bvh_node; /* leaf: count > 0 */

typedef struct {
    int64_t n_tris, n_sph, n_prims;
    double* tv;          /* [n_tris][9] fp64 vertices (exact widening of the fp32 input) */
    uint32_t* tmat;
    double* sp;          /* [n_sph][4] centre, radius */
    uint32_t* smat;
    in_mat* mats;
    int32_t n_mats;
    in_cam cam;
    bvh_node* nodes;
    int64_t n_nodes;
    int64_t* order;      /* prim ids in leaf order */
} orc_scene;

static box3 prim_box(const orc_scene* sc, int64_t id) {
    box3 b;
    if (id < sc->n_tris) {
        const double* v = sc->tv + 9 * id;
        for (int a = 0; a < 3; ++a) {
            double lo = v[a], hi = v[a];
            if (v[3 + a] < lo) lo = v[3 + a];
            if (v[6 + a] < lo) lo = v[6 + a];
            if (v[3 + a] > hi) hi = v[3 + a];
            if (v[6 + a] > hi) hi = v[6 + a];
            b.lo[a] = lo; b.hi[a] = hi;
        }
    } else {
        const double* s = sc->sp + 4 * (id - sc->n_tris);
        for (int a = 0; a < 3; ++a) {
            /* rounded outward so the box always contains the exact sphere */
            b.lo[a] = nextafter(s[a] - s[3], -INFINITY);
            b.hi[a] = nextafter(s[a] + s[3], INFINITY);
        }
    }
    return b;
}

static void box_empty(box3* b) {
    for (int a = 0; a < 3; ++a) { b->lo[a] = INFINITY; b->hi[a] = -INFINITY; }
}
static void box_grow(box3* b, const box3* o) {
    for (int a = 0; a < 3; ++a) {
        if (o->lo[a] < b->lo[a]) b->lo[a] = o->lo[a];
        if (o->hi[a] > b->hi[a]) b->hi[a] = o->hi[a];
    }
}
static double box_area(const box3* b) {
    double dx = b->hi[0] - b->lo[0], dy = b->hi[1] - b->lo[1], dz = b->hi[2] - b->lo[2];
    if (dx < 0) return 0.0;
    return 2.0 * (dx * dy + dy * dz + dz * dx);
}

typedef struct { int64_t node, first, count; } build_item;

static void build_bvh(orc_scene* sc) {
    int64_t n = sc->n_prims;
    sc->order = (int64_t*)malloc(sizeof(int64_t) * (n > 0 ? n : 1));
    box3* pb = (box3*)malloc(sizeof(box3) * (n > 0 ? n : 1));
    double* cen = (double*)malloc(sizeof(double) * 3 * (n > 0 ? n : 1));
    for (int64_t i = 0; i < n; ++i) {
        sc->order[i] = i;
        pb[i] = prim_box(sc, i);
        for (int a = 0; a < 3; ++a) cen[3 * i + a] = 0.5 * (pb[i].lo[a] + pb[i].hi[a]);
    }
    int64_t cap = 2 * n + 1;
    sc->nodes = (bvh_node*)malloc(sizeof(bvh_node) * cap);
    sc->n_nodes = 0;
    if (n == 0) { free(pb); free(cen); return; }
    build_item* stack = (build_item*)malloc(sizeof(build_item) * 1024);
    int sp = 0;
    sc->n_nodes = 1;
    stack[sp++] = (build_item){0, 0, n};
    enum { NB = 16 };
    while (sp > 0) {
        build_item it = stack[--sp];
        bvh_node* nd = &sc->nodes[it.node];
        box3 bb, cb;
        box_empty(&bb); box_empty(&cb);
        for (int64_t i = it.first; i < it.first + it.count; ++i) {
            int64_t id = sc->order[i];
            box_grow(&bb, &pb[id]);
            box3 c; for (int a = 0; a < 3; ++a) c.lo[a] = c.hi[a] = cen[3 * id + a];
            box_grow(&cb, &c);
        }
        nd->b = bb;
        int axis = 0;
        double ext = cb.hi[0] - cb.lo[0];
        for (int a = 1; a < 3; ++a) if (cb.hi[a] - cb.lo[a] > ext) { ext = cb.hi[a] - cb.lo[a]; axis = a; }
        int64_t split = -1;
        if (it.count > 2 && ext > 0.0) {
            int64_t cnt[NB] = {0};
            box3 bins[NB];
            for (int k = 0; k < NB; ++k) box_empty(&bins[k]);
            double scale = NB / ext;
            for (int64_t i = it.first; i < it.first + it.count; ++i) {
                int64_t id = sc->order[i];
                int k = (int)((cen[3 * id + axis] - cb.lo[axis]) * scale);
                if (k >= NB) k = NB - 1;
                if (k < 0) k = 0;
                cnt[k]++;
                box_grow(&bins[k], &pb[id]);
            }
            double best = INFINITY; int best_k = -1;
            for (int k = 0; k < NB - 1; ++k) {
                box3 l, r; box_empty(&l); box_empty(&r);
                int64_t nl = 0, nr = 0;
                for (int j = 0; j <= k; ++j) { box_grow(&l, &bins[j]); nl += cnt[j]; }
                for (int j = k + 1; j < NB; ++j) { box_grow(&r, &bins[j]); nr += cnt[j]; }
                if (nl == 0 || nr == 0) continue;
                double c = box_area(&l) * (double)nl + box_area(&r) * (double)nr;
                if (c < best) { best = c; best_k = k; }
            }
            double leaf_cost = box_area(&bb) * (double)it.count;
            if (best_k >= 0 && (best < leaf_cost || it.count > 4)) {
                /* partition by bin index */
                int64_t i = it.first, j = it.first + it.count - 1;
                while (i <= j) {
                    int64_t id = sc->order[i];
                    int k = (int)((cen[3 * id + axis] - cb.lo[axis]) * scale);
                    if (k >= NB) k = NB - 1;
                    if (k < 0) k = 0;
                    if (k <= best_k) ++i;
                    else { int64_t t = sc->order[i]; sc->order[i] = sc->order[j]; sc->order[j] = t; --j; }
                }
                split = i;
            }
        } else if (it.count > 4) {
            split = it.first + it.count / 2;  /* coincident centroids: median split keeps leaves small */
        }
        if (split > it.first && split < it.first + it.count) {
            int64_t l = sc->n_nodes++, r = sc->n_nodes++;
            nd = &sc->nodes[it.node];
            nd->left = (int32_t)l; nd->right = (int32_t)r; nd->first = 0; nd->count = 0;
            stack[sp++] = (build_item){r, split, it.first + it.count - split};
            stack[sp++] = (build_item){l, it.first, split - it.first};
        } else {
            nd->left = nd->right = -1;
            nd->first = (int32_t)it.first; nd->count = (int32_t)it.count;
        }
    }
    free(stack); free(pb); free(cen);
}

EXPORT orc_scene* orc_scene_create(const in_tri* tris, int64_t n_tris, const in_sphere* sph, int64_t n_sph,
                                   const in_mat* mats, int32_t n_mats, const in_cam* cam) {
    orc_scene* sc = (orc_scene*)calloc(1, sizeof(orc_scene));
    sc->n_tris = n_tris; sc->n_sph = n_sph; sc->n_prims = n_tris + n_sph;
    sc->tv = (double*)malloc(sizeof(double) * 9 * (n_tris > 0 ? n_tris : 1));
    sc->tmat = (uint32_t*)malloc(sizeof(uint32_t) * (n_tris > 0 ? n_tris : 1));
    for (int64_t i = 0; i < n_tris; ++i) {
        for (int a = 0; a < 3; ++a) {
            sc->tv[9 * i + a] = tris[i].v0[a];
            sc->tv[9 * i + 3 + a] = tris[i].v1[a];
            sc->tv[9 * i + 6 + a] = tris[i].v2[a];
        }
        sc->tmat[i] = tris[i].material;
    }
    sc->sp = (double*)malloc(sizeof(double) * 4 * (n_sph > 0 ? n_sph : 1));
    sc->smat = (uint32_t*)malloc(sizeof(uint32_t) * (n_sph > 0 ? n_sph : 1));
    for (int64_t i = 0; i < n_sph; ++i) {
        for (int a = 0; a < 3; ++a) sc->sp[4 * i + a] = sph[i].c[a];
        sc->sp[4 * i + 3] = sph[i].r;
        sc->smat[i] = sph[i].material;
    }
    sc->mats = (in_mat*)malloc(sizeof(in_mat) * (n_mats > 0 ? n_mats : 1));
    memcpy(sc->mats, mats, sizeof(in_mat) * n_mats);
    sc->n_mats = n_mats;
    sc->cam = *cam;
    build_bvh(sc);
    return sc;
}

EXPORT void orc_scene_destroy(orc_scene* sc) {
    if (!sc) return;
    free(sc->tv); free(sc->tmat); free(sc->sp); free(sc->smat); free(sc->mats);
    free(sc->nodes); free(sc->order); free(sc);
}

EXPORT int64_t orc_scene_n_nodes(const orc_scene* sc) { return sc->n_nodes; }

/* ---------------------------------------------------------------------------------------------- */
/* Intersection (fp64)                                                                              */
/* ---------------------------------------------------------------------------------------------- */
typedef struct { int kx, ky, kz; double Sx, Sy, Sz; double o[3], d[3], inv[3]; } ray_pre;

static void ray_prepare(const double o[3], const double d[3], ray_pre* r) {
    /* Woop et al. 2013, Sec. 3: kz = dimension of largest |d| (first on ties), kx, ky follow; swap to
       keep winding when d[kz] < 0; shear constants S. */
    int kz = 0;
    if (fabs(d[1]) > fabs(d[kz])) kz = 1;
    if (fabs(d[2]) > fabs(d[kz])) kz = 2;
    int kx = kz + 1; if (kx == 3) kx = 0;
    int ky = kx + 1; if (ky == 3) ky = 0;
    if (d[kz] < 0.0) { int t = kx; kx = ky; ky = t; }
    r->kx = kx; r->ky = ky; r->kz = kz;
    r->Sx = d[kx] / d[kz];
    r->Sy = d[ky] / d[kz];
    r->Sz = 1.0 / d[kz];
    for (int a = 0; a < 3; ++a) { r->o[a] = o[a]; r->d[a] = d[a]; r->inv[a] = 1.0 / d[a]; }
}

/* Watertight ray/triangle test (Woop, Benthin, Wald, JCGT 2013; PBRT-v3 Sec. 3.6.2), fp64.
   Returns 1 with t > 0, barycentrics (b0, b1, b2) = (U, V, W)/det; 0 otherwise. */
static int tri_test(const ray_pre* r, const double* v, double* t_out, double bary[3]) {
    double A[3], B[3], C[3];
    for (int a = 0; a < 3; ++a) { A[a] = v[a] - r->o[a]; B[a] = v[3 + a] - r->o[a]; C[a] = v[6 + a] - r->o[a]; }
    const int kx = r->kx, ky = r->ky, kz = r->kz;
    double Ax = A[kx] - r->Sx * A[kz];
    double Ay = A[ky] - r->Sy * A[kz];
    double Bx = B[kx] - r->Sx * B[kz];
    double By = B[ky] - r->Sy * B[kz];
    double Cx = C[kx] - r->Sx * C[kz];
    double Cy = C[ky] - r->Sy * C[kz];
    double U = Cx * By - Cy * Bx;
    double V = Ax * Cy - Ay * Cx;
    double W = Bx * Ay - By * Ax;
    if ((U < 0.0 || V < 0.0 || W < 0.0) && (U > 0.0 || V > 0.0 || W > 0.0)) return 0;
    double det = (U + V) + W;
    if (det == 0.0) return 0;
    double Az = r->Sz * A[kz];
    double Bz = r->Sz * B[kz];
    double Cz = r->Sz * C[kz];
    double T = (U * Az + V * Bz) + W * Cz;
    if (det < 0.0 && T >= 0.0) return 0;
    if (det > 0.0 && T <= 0.0) return 0;
    *t_out = T / det;
    bary[0] = U / det; bary[1] = V / det; bary[2] = W / det;
    return 1;
}

/* Ray/sphere: |o + t d - c|^2 = r^2, smaller positive root (reading R12), fp64.
   graze = 1 - (d_perp / r)^2 = disc / (a r^2), the near-tangent measure used by the hit gate. */
static int sph_test(const ray_pre* r, const double* s, double* t_out, double* graze) {
    double oc[3] = {r->o[0] - s[0], r->o[1] - s[1], r->o[2] - s[2]};
    double a = (r->d[0] * r->d[0] + r->d[1] * r->d[1]) + r->d[2] * r->d[2];
    double b = (oc[0] * r->d[0] + oc[1] * r->d[1]) + oc[2] * r->d[2];
    double c = ((oc[0] * oc[0] + oc[1] * oc[1]) + oc[2] * oc[2]) - s[3] * s[3];
    double disc = b * b - a * c;
    if (disc < 0.0) return 0;
    double sq = sqrt(disc);
    double t0 = (-b - sq) / a;
    double t1 = (-b + sq) / a;
    double t;
    if (t0 > 0.0) t = t0;
    else if (t1 > 0.0) t = t1;
    else return 0;
    *t_out = t;
    *graze = disc / (a * (s[3] * s[3]));
    return 1;
}

typedef struct { int64_t prim; double t; double bary[3]; double edge; } hit_rec; /* prim -1 = miss */

/* closer in (t, id) lexicographic order (reading R11) */
static int closer(double t, int64_t id, const hit_rec* h) {
    return h->prim < 0 || t < h->t || (t == h->t && id < h->prim);
}

static void test_prim(const orc_scene* sc, const ray_pre* r, int64_t id, hit_rec* h) {
    double t, bary[3], g;
    if (id < sc->n_tris) {
        if (tri_test(r, sc->tv + 9 * id, &t, bary) && closer(t, id, h)) {
            h->prim = id; h->t = t;
            h->bary[0] = bary[0]; h->bary[1] = bary[1]; h->bary[2] = bary[2];
            double m = bary[0]; if (bary[1] < m) m = bary[1]; if (bary[2] < m) m = bary[2];
            h->edge = m;
        }
    } else {
        if (sph_test(r, sc->sp + 4 * (id - sc->n_tris), &t, &g) && closer(t, id, h)) {
            h->prim = id; h->t = t; h->bary[0] = h->bary[1] = h->bary[2] = 0.0; h->edge = g;
        }
    }
}

static void closest_brute(const orc_scene* sc, const ray_pre* r, hit_rec* h) {
    h->prim = -1;
    for (int64_t id = 0; id < sc->n_prims; ++id) test_prim(sc, r, id, h);
}

/* robust slab test: PBRT-v3 Sec. 3.9.2 (t_far scaled by 1 + 2 gamma_3); zero direction handled
   explicitly. Returns entry distance (>= 0 clamp not applied) or +inf on miss. */
static double slab(const ray_pre* r, const box3* b, double t_max) {
    const double g3 = 3.0 * 0x1p-53 / (1.0 - 3.0 * 0x1p-53);
    double t0 = 0.0, t1 = t_max;
    for (int a = 0; a < 3; ++a) {
        if (r->d[a] == 0.0) {
            if (r->o[a] < b->lo[a] || r->o[a] > b->hi[a]) return INFINITY;
            continue;
        }
        double tn = (b->lo[a] - r->o[a]) * r->inv[a];
        double tf = (b->hi[a] - r->o[a]) * r->inv[a];
        if (tn > tf) { double t = tn; tn = tf; tf = t; }
        tf *= 1.0 + 2.0 * g3;
        if (tn > t0) t0 = tn;
        if (tf < t1) t1 = tf;
        if (t0 > t1) return INFINITY;
    }
    return t0;
}

static void closest_bvh(const orc_scene* sc, const ray_pre* r, hit_rec* h) {
    h->prim = -1;
    if (sc->n_nodes == 0) return;
    int32_t stack[1024];
    int sp = 0;
    stack[sp++] = 0;
    while (sp > 0) {
        int32_t ni = stack[--sp];
        const bvh_node* nd = &sc->nodes[ni];
        /* cull only boxes entered beyond the best hit: ties are kept (reading R11). The entry distance
           carries its own rounding (and the primitive's t its own), so a box whose computed entry lies a
           few ulps beyond a tied hit at its face can still hold an equal-t, smaller-id primitive (rays
           through a shared vertex): the bound is widened by 2^-32 relative, far above the fp64 rounding of
           both, so the BVH returns exactly the brute-force (t, id) minimum. */
        double tb = h->prim < 0 ? INFINITY : h->t * (1.0 + 0x1p-32);
        double te = slab(r, &nd->b, INFINITY);
        if (te == INFINITY || te > tb) continue;
        if (nd->count > 0) {
            for (int64_t i = nd->first; i < nd->first + nd->count; ++i) test_prim(sc, r, sc->order[i], h);
        } else {
            stack[sp++] = nd->right;
            stack[sp++] = nd->left;
        }
    }
}

EXPORT void orc_closest_hit(const orc_scene* sc, const double* o, const double* d, int64_t n, int brute,
                            int64_t* prim, double* t, double* bary, double* edge) {
    for (int64_t i = 0; i < n; ++i) {
        ray_pre r;
        ray_prepare(o + 3 * i, d + 3 * i, &r);
        hit_rec h;
        if (brute) closest_brute(sc, &r, &h); else closest_bvh(sc, &r, &h);
        prim[i] = h.prim;
        t[i] = h.prim >= 0 ? h.t : INFINITY;
        for (int a = 0; a < 3; ++a) bary[3 * i + a] = h.prim >= 0 ? h.bary[a] : 0.0;
        edge[i] = h.prim >= 0 ? h.edge : 0.0;
    }
}

/* ---------------------------------------------------------------------------------------------- */
/* Camera (IEEE fp32, reading R22)                                                                  */
/* ---------------------------------------------------------------------------------------------- */
typedef struct { float f[3], r[3], u[3], eye[3]; float ta, t; } cam32;

static void cam_setup(const in_cam* c, int32_t W, int32_t H, cam32* k) {
    double f[3], r[3], u[3];
    for (int a = 0; a < 3; ++a) f[a] = (double)c->look_at[a] - (double)c->eye[a];
    double lf = sqrt(f[0] * f[0] + f[1] * f[1] + f[2] * f[2]);
    for (int a = 0; a < 3; ++a) f[a] /= lf;
    double up[3] = {c->up[0], c->up[1], c->up[2]};
    r[0] = f[1] * up[2] - f[2] * up[1];
    r[1] = f[2] * up[0] - f[0] * up[2];
    r[2] = f[0] * up[1] - f[1] * up[0];
    double lr = sqrt(r[0] * r[0] + r[1] * r[1] + r[2] * r[2]);
    for (int a = 0; a < 3; ++a) r[a] /= lr;
    u[0] = r[1] * f[2] - r[2] * f[1];
    u[1] = r[2] * f[0] - r[0] * f[2];
    u[2] = r[0] * f[1] - r[1] * f[0];
    double t = tan(0.5 * (double)c->vfov_deg * 3.14159265358979323846 / 180.0);
    for (int a = 0; a < 3; ++a) { k->f[a] = (float)f[a]; k->r[a] = (float)r[a]; k->u[a] = (float)u[a]; k->eye[a] = c->eye[a]; }
    k->ta = (float)(t * ((double)W / (double)H));
    k->t = (float)t;
}

/* d = normalize(f + sx*ta*r + sy*t*u), sx = 2(x+xi0)/W - 1, sy = 1 - 2(y+xi1)/H, left to right,
   each operation a separately rounded fp32 op (this file is compiled with -ffp-contract=off). */
static void cam_dir32(const cam32* k, int32_t W, int32_t H, int32_t x, int32_t y, float xi0, float xi1, float d[3]) {
    float px = (float)x + xi0;
    float py = (float)y + xi1;
    float sx = (2.0f * px) / (float)W - 1.0f;
    float sy = 1.0f - (2.0f * py) / (float)H;
    float cx = sx * k->ta;
    float cy = sy * k->t;
    float v[3];
    for (int a = 0; a < 3; ++a) {
        float m1 = cx * k->r[a];
        float s1 = k->f[a] + m1;
        float m2 = cy * k->u[a];
        v[a] = s1 + m2;
    }
    float l2 = (v[0] * v[0] + v[1] * v[1]) + v[2] * v[2];
    float l = sqrtf(l2);
    for (int a = 0; a < 3; ++a) d[a] = v[a] / l;
}

EXPORT void orc_camera_dir(const in_cam* cam, int32_t W, int32_t H, int32_t x, int32_t y, float xi0, float xi1,
                           float* d) {
    cam32 k;
    cam_setup(cam, W, H, &k);
    cam_dir32(&k, W, H, x, y, xi0, xi1, d);
}

EXPORT void orc_camera_rays(const in_cam* cam, int32_t W, int32_t H, uint64_t seed, int32_t sample,
                            const int64_t* pix, int64_t n, float* dirs /* [n][3] */) {
    cam32 k;
    cam_setup(cam, W, H, &k);
    for (int64_t i = 0; i < n; ++i) {
        double u[4];
        int64_t p = pix[i];
        draw4(seed, (uint32_t)p, (uint32_t)sample, 0u, u);
        cam_dir32(&k, W, H, (int32_t)(p % W), (int32_t)(p / W), (float)u[0], (float)u[1], dirs + 3 * i);
    }
}

/* ---------------------------------------------------------------------------------------------- */
/* Equirect map (SPEC.md:438 convention) and HDR-NIF (SIREN per BASELINE.json)        */
/* ---------------------------------------------------------------------------------------------- */
static void equirect(const double d[3], double* u, double* v) {
    const double PI = 3.14159265358979323846;
    double len = sqrt((d[0] * d[0] + d[1] * d[1]) + d[2] * d[2]);
    double uu;
    if (d[0] == 0.0 && d[2] == 0.0) uu = 0.5;
    else {
        uu = 0.5 + atan2(d[0], -d[2]) / (2.0 * PI);
        if (uu >= 1.0) uu -= 1.0;
    }
    double y = d[1] / len;
    if (y > 1.0) y = 1.0;
    if (y < -1.0) y = -1.0;
    *u = uu;
    *v = acos(y) / PI;
}

EXPORT void orc_equirect(const double* d, int64_t n, double* uv) {
    for (int64_t i = 0; i < n; ++i) equirect(d + 3 * i, uv + 2 * i, uv + 2 * i + 1);
}

typedef struct { double* W[5]; double* b[5]; } nif64;
static const int NIF_IN[5] = {2, 128, 128, 128, 128};
static const int NIF_OUT[5] = {128, 128, 128, 128, 3};

static double half_to_double(uint16_t h) {
    int s = (h >> 15) & 1, e = (h >> 10) & 31, m = h & 1023;
    double v;
    if (e == 0) v = ldexp((double)m, -24);
    else if (e == 31) v = m ? NAN : INFINITY;
    else v = ldexp((double)(m | 1024), e - 25);
    return s ? -v : v;
}

static void nif_unpack(const uint16_t* blob, nif64* n) {
    int64_t off = 0;
    for (int l = 0; l < 5; ++l) {
        int fi = NIF_IN[l], fo = NIF_OUT[l];
        n->W[l] = (double*)malloc(sizeof(double) * fi * fo);
        n->b[l] = (double*)malloc(sizeof(double) * fo);
        for (int i = 0; i < fi * fo; ++i) n->W[l][i] = half_to_double(blob[off++]);
        for (int i = 0; i < fo; ++i) n->b[l][i] = half_to_double(blob[off++]);
    }
}
static void nif_free(nif64* n) { for (int l = 0; l < 5; ++l) { free(n->W[l]); free(n->b[l]); } }

/* x0 = (2u-1, 2v-1); h1 = sin(W1 x0 + b1); h_{k+1} = sin(W_{k+1} h_k + b_{k+1}), k=1..3;
   y = W5 h4 + b5 (log-RGB). Weights are the fp16 blob widened exactly (w0 already folded). */
static void nif_eval(const nif64* n, double u, double v, double y[3]) {
    double a[128], h[128];
    a[0] = 2.0 * u - 1.0; a[1] = 2.0 * v - 1.0;
    for (int l = 0; l < 4; ++l) {
        int fi = NIF_IN[l], fo = NIF_OUT[l];
        for (int o = 0; o < fo; ++o) {
            double s = 0.0;
            for (int i = 0; i < fi; ++i) s += n->W[l][o * fi + i] * a[i];
            h[o] = sin(s + n->b[l][o]);
        }
        memcpy(a, h, sizeof(double) * fo);
    }
    for (int o = 0; o < 3; ++o) {
        double s = 0.0;
        for (int i = 0; i < 128; ++i) s += n->W[4][o * 128 + i] * a[i];
        y[o] = s + n->b[4][o];
    }
}

EXPORT void orc_nif_eval(const uint16_t* blob, const double* uv, int64_t n, double* y_out) {
    nif64 net;
    nif_unpack(blob, &net);
    for (int64_t i = 0; i < n; ++i) nif_eval(&net, uv[2 * i], uv[2 * i + 1], y_out + 3 * i);
    nif_free(&net);
}

/* The paper's own NIF (reading R4): Fourier features of x = (u, v),
   gamma = [sin(2 pi B x) (20), cos(2 pi B x) (20)]; h0 = relu(W0 gamma + b0) (128); h1 = relu(W1 h0 + b1)
   (88); h2 = relu(W2 [h1, gamma] + b2) (concat skip, 128); h3 = relu(W3 h2 + b3); yuv = W4 h3 + b4;
   rgb_log = M yuv with M the fixed BT.601 YUV->RGB matrix. Returns rgb_log (the env is exp). */
static const int FR_IN[5] = {40, 128, 128, 128, 128};
static const int FR_OUT[5] = {128, 88, 128, 128, 3};

static void fr_eval(const double* B, double* const W[5], double* const b[5], double u, double v, double y[3]) {
    const double PI = 3.14159265358979323846;
    double g[40], a[128], h[128];
    for (int j = 0; j < 20; ++j) {
        double p = 2.0 * PI * (B[2 * j] * u + B[2 * j + 1] * v);
        g[j] = sin(p);
        g[20 + j] = cos(p);
    }
    memcpy(a, g, sizeof(double) * 40);
    for (int l = 0; l < 4; ++l) {
        int fi = FR_IN[l], fo = FR_OUT[l];
        for (int o = 0; o < fo; ++o) {
            double s = 0.0;
            for (int i = 0; i < fi; ++i) s += W[l][o * fi + i] * a[i];
            s += b[l][o];
            h[o] = s > 0.0 ? s : 0.0;
        }
        if (l == 1) {                     /* concat skip: [h1 (88), gamma (40)] */
            memcpy(a, h, sizeof(double) * 88);
            memcpy(a + 88, g, sizeof(double) * 40);
        } else {
            memcpy(a, h, sizeof(double) * fo);
        }
    }
    double yuv[3];
    for (int o = 0; o < 3; ++o) {
        double s = 0.0;
        for (int i = 0; i < 128; ++i) s += W[4][o * 128 + i] * a[i];
        yuv[o] = s + b[4][o];
    }
    y[0] = yuv[0] + 1.13983 * yuv[2];
    y[1] = yuv[0] - 0.39465 * yuv[1] - 0.58060 * yuv[2];
    y[2] = yuv[0] + 2.03211 * yuv[1];
}

EXPORT void orc_fr_eval(const uint16_t* blob, const double* uv, int64_t n, double* y_out) {
    double B[40];
    double* W[5];
    double* b[5];
    int64_t off = 0;
    for (int i = 0; i < 40; ++i) B[i] = half_to_double(blob[off++]);
    for (int l = 0; l < 5; ++l) {
        W[l] = (double*)malloc(sizeof(double) * FR_IN[l] * FR_OUT[l]);
        b[l] = (double*)malloc(sizeof(double) * FR_OUT[l]);
        for (int i = 0; i < FR_IN[l] * FR_OUT[l]; ++i) W[l][i] = half_to_double(blob[off++]);
        for (int i = 0; i < FR_OUT[l]; ++i) b[l][i] = half_to_double(blob[off++]);
    }
    for (int64_t i = 0; i < n; ++i) fr_eval(B, W, b, uv[2 * i], uv[2 * i + 1], y_out + 3 * i);
    for (int l = 0; l < 5; ++l) { free(W[l]); free(b[l]); }
}

/* The paper's NIF family of the size sweep ("hidden size H (128) and number of dense-relu
   layers L (4) can be varied"; Fig. nrf-vs-blender H64 L2 / H256 L4 / H1024 L8, PAPER.md:225-227;
   DESIGN.md reading R23): 40 Fourier features -> L dense ReLU layers of width H, where layer c =
   the largest odd index below L/2 (c = 0 when there is none, L <= 2) outputs H - 40 units and is
   concatenated with the 40 features ("always concatenated with the last odd layer before the middle
   of the network, which has a reduced dense layer output size to compensate") -> linear H -> 3 (YUV,
   log) -> fixed BT.601 YUV -> RGB. Blob: B [20][2], then W_l [out][in], b_l [out] for the L + 1
   layers. (H, L) = (128, 4) is the network of orc_fr_eval. */
EXPORT int orc_fr_concat_layer(int32_t L) {
    int c = 0;
    for (int l = 1; 2 * l < L; l += 2) c = l;
    return c;
}

EXPORT void orc_fr_dims(int32_t H, int32_t L, int32_t* fin, int32_t* fout) {
    const int c = orc_fr_concat_layer(L);
    for (int l = 0; l <= L; ++l) {
        fin[l] = l == 0 ? 40 : H;
        fout[l] = l == L ? 3 : (l == c ? H - 40 : H);
    }
}

typedef struct {
    int H, L, c;
    int32_t fin[17], fout[17];
    double B[40];
    double* W[17];
    double* b[17];
} fr_net;

static void fr_unpack(int32_t H, int32_t L, const uint16_t* blob, fr_net* n) {
    n->H = H; n->L = L; n->c = orc_fr_concat_layer(L);
    orc_fr_dims(H, L, n->fin, n->fout);
    int64_t off = 0;
    for (int i = 0; i < 40; ++i) n->B[i] = half_to_double(blob[off++]);
    for (int l = 0; l <= L; ++l) {
        n->W[l] = (double*)malloc(sizeof(double) * n->fin[l] * n->fout[l]);
        n->b[l] = (double*)malloc(sizeof(double) * n->fout[l]);
        for (int64_t i = 0; i < (int64_t)n->fin[l] * n->fout[l]; ++i) n->W[l][i] = half_to_double(blob[off++]);
        for (int i = 0; i < n->fout[l]; ++i) n->b[l][i] = half_to_double(blob[off++]);
    }
}

static void fr_net_free(fr_net* n) {
    for (int l = 0; l <= n->L; ++l) { free(n->W[l]); free(n->b[l]); }
}

/* RGB log radiance of (u, v), the steps in the order of the comment above */
static void fr_net_eval(const fr_net* n, double u, double v, double y[3]) {
    const double PI = 3.14159265358979323846;
    const int H = n->H, L = n->L;
    double g[40], a[1024], h[1024];
    for (int j = 0; j < 20; ++j) {
        const double p = 2.0 * PI * (n->B[2 * j] * u + n->B[2 * j + 1] * v);
        g[j] = sin(p);
        g[20 + j] = cos(p);
    }
    memcpy(a, g, sizeof(double) * 40);
    for (int l = 0; l < L; ++l) {
        for (int o = 0; o < n->fout[l]; ++o) {
            double s = 0.0;
            for (int i = 0; i < n->fin[l]; ++i) s += n->W[l][(int64_t)o * n->fin[l] + i] * a[i];
            s += n->b[l][o];
            h[o] = s > 0.0 ? s : 0.0;
        }
        memcpy(a, h, sizeof(double) * n->fout[l]);
        if (l == n->c) memcpy(a + (H - 40), g, sizeof(double) * 40);   /* concat skip: [h_c, gamma] */
    }
    double yuv[3];
    for (int o = 0; o < 3; ++o) {
        double s = 0.0;
        for (int i = 0; i < H; ++i) s += n->W[L][(int64_t)o * H + i] * a[i];
        yuv[o] = s + n->b[L][o];
    }
    y[0] = yuv[0] + 1.13983 * yuv[2];
    y[1] = yuv[0] - 0.39465 * yuv[1] - 0.58060 * yuv[2];
    y[2] = yuv[0] + 2.03211 * yuv[1];
}

/* OCP e4m3 (1 sign, 4 exponent bits with bias 7, 3 mantissa bits, no infinities, largest finite 448):
   round to nearest, ties to the even code, saturating -- written as a search over the decoded table of
   the 127 non-negative finite codes, independent of the CUDA path's arithmetic conversion. */
static double e4m3_value(int code) {          /* 0 <= code <= 0x7E */
    const int e = code >> 3, m = code & 7;
    return e == 0 ? ldexp((double)m, -9) : ldexp((double)(8 + m), e - 10);
}
static double e4m3_round(double x) {
    double a = fabs(x);
    if (a >= 448.0) a = 448.0;
    int lo = 0, hi = 0x7E;                     /* largest code with value <= a */
    while (lo < hi) {
        const int mid = (lo + hi + 1) / 2;
        if (e4m3_value(mid) <= a) lo = mid; else hi = mid - 1;
    }
    double r = e4m3_value(lo);
    if (lo < 0x7E && r < a) {
        const double up = e4m3_value(lo + 1);
        if (up - a < a - r || (up - a == a - r && ((lo + 1) & 1) == 0)) r = up;
    }
    return x < 0 ? -r : r;
}
EXPORT double orc_e4m3_round(double x) { return e4m3_round(x); }

/* The fp8 variant (PT_NIF_FP8, reading R24): weights rounded to e4m3 once (fr_quantize_fp8),
   the features and every hidden activation rounded to e4m3 before they feed the next layer; biases,
   sums and the output in fp64. */
static void fr_quantize_fp8(fr_net* net) {
    for (int l = 0; l <= net->L; ++l)
        for (int64_t i = 0; i < (int64_t)net->fin[l] * net->fout[l]; ++i) net->W[l][i] = e4m3_round(net->W[l][i]);
}
static void fr_net_eval_fp8(const fr_net* net, double u, double v, double y[3]) {
    const double PI = 3.14159265358979323846;
    const int H = net->H, L = net->L;
    double g[40], a[1024], h[1024];
    for (int j = 0; j < 20; ++j) {
        const double p = 2.0 * PI * (net->B[2 * j] * u + net->B[2 * j + 1] * v);
        g[j] = e4m3_round(sin(p));
        g[20 + j] = e4m3_round(cos(p));
    }
    memcpy(a, g, sizeof(double) * 40);
    for (int l = 0; l < L; ++l) {
        for (int o = 0; o < net->fout[l]; ++o) {
            double s = 0.0;
            for (int i = 0; i < net->fin[l]; ++i) s += net->W[l][(int64_t)o * net->fin[l] + i] * a[i];
            s += net->b[l][o];
            h[o] = e4m3_round(s > 0.0 ? s : 0.0);
        }
        memcpy(a, h, sizeof(double) * net->fout[l]);
        if (l == net->c) memcpy(a + (H - 40), g, sizeof(double) * 40);
    }
    double yuv[3];
    for (int o = 0; o < 3; ++o) {
        double s = 0.0;
        for (int i = 0; i < H; ++i) s += net->W[L][(int64_t)o * H + i] * a[i];
        yuv[o] = s + net->b[L][o];
    }
    y[0] = yuv[0] + 1.13983 * yuv[2];
    y[1] = yuv[0] - 0.39465 * yuv[1] - 0.58060 * yuv[2];
    y[2] = yuv[0] + 2.03211 * yuv[1];
}
EXPORT void orc_fr_eval_hl_fp8(int32_t H, int32_t L, const uint16_t* blob, const double* uv, int64_t n, double* y_out) {
    fr_net net;
    fr_unpack(H, L, blob, &net);
    fr_quantize_fp8(&net);
    for (int64_t q = 0; q < n; ++q) fr_net_eval_fp8(&net, uv[2 * q], uv[2 * q + 1], y_out + 3 * q);
    fr_net_free(&net);
}

EXPORT void orc_fr_eval_hl(int32_t H, int32_t L, const uint16_t* blob, const double* uv, int64_t n, double* y_out) {
    fr_net net;
    fr_unpack(H, L, blob, &net);
    for (int64_t q = 0; q < n; ++q) fr_net_eval(&net, uv[2 * q], uv[2 * q + 1], y_out + 3 * q);
    fr_net_free(&net);
}

/* ---------------------------------------------------------------------------------------------- */
/* Scattering (readings R9, R10)                                        */
/* ---------------------------------------------------------------------------------------------- */
static double dot3(const double a[3], const double b[3]) { return (a[0] * b[0] + a[1] * b[1]) + a[2] * b[2]; }
static void normalize3(double v[3]) {
    double l = sqrt(dot3(v, v));
    v[0] /= l; v[1] /= l; v[2] /= l;
}

/* Lambertian: cosine-weighted hemisphere about n with the branchless ONB of Duff et al. (JCGT 2017). */
static void scatter_lambert(const double n[3], double xi0, double xi1, double wi[3]) {
    const double PI = 3.14159265358979323846;
    double s = copysign(1.0, n[2]);
    double a = -1.0 / (s + n[2]);
    double b = n[0] * n[1] * a;
    double t1[3] = {1.0 + s * n[0] * n[0] * a, s * b, -s * n[0]};
    double t2[3] = {b, s + n[1] * n[1] * a, -n[1]};
    double rho = sqrt(xi0), phi = 2.0 * PI * xi1;
    double c1 = rho * cos(phi), c2 = rho * sin(phi), c3 = sqrt(1.0 - xi0);
    for (int k = 0; k < 3; ++k) wi[k] = (c1 * t1[k] + c2 * t2[k]) + c3 * n[k];
}

static void scatter_mirror(const double d[3], const double n[3], double wi[3]) {
    double dn = dot3(d, n);
    for (int k = 0; k < 3; ++k) wi[k] = d[k] - 2.0 * dn * n[k];
}

/* Dielectric (Schlick Fresnel, TIR -> F = 1). Returns +1 when reflected (leaves on the n side),
   -1 when refracted (leaves on the -n side). n faces the incoming ray; entering iff d.n_g < 0. */
static int scatter_dielectric(const double d[3], const double n[3], int entering, double ior, double xi2,
                              double wi[3], double* F_out) {
    double eta = entering ? 1.0 / ior : ior;
    double cosi = -dot3(d, n);
    double sin2t = eta * eta * (1.0 - cosi * cosi);
    double F, cost = 0.0;
    if (sin2t > 1.0) F = 1.0;
    else {
        cost = sqrt(1.0 - sin2t);
        double c = entering ? cosi : cost;
        double r0 = (1.0 - ior) / (1.0 + ior);
        r0 = r0 * r0;
        double m = 1.0 - c;
        F = r0 + (1.0 - r0) * (m * m * m * m * m);
    }
    *F_out = F;
    if (xi2 < F) {
        for (int k = 0; k < 3; ++k) wi[k] = d[k] + 2.0 * cosi * n[k];
        return 1;
    }
    for (int k = 0; k < 3; ++k) wi[k] = eta * d[k] + (eta * cosi - cost) * n[k];
    return -1;
}

EXPORT void orc_scatter(int kind, const double* d, const double* ng, double ior, const double* xi,
                        double* wi_out, double* F_out, int32_t* side_out) {
    /* one scatter event for pin tests; same code path as the renderer */
    double n[3];
    int entering = dot3(d, ng) < 0.0;
    for (int k = 0; k < 3; ++k) n[k] = entering ? ng[k] : -ng[k];
    double wi[3]; int side = 1; double F = 0.0;
    if (kind == K_LAMBERT) scatter_lambert(n, xi[0], xi[1], wi);
    else if (kind == K_MIRROR) scatter_mirror(d, n, wi);
    else side = scatter_dielectric(d, n, entering, ior, xi[2], wi, &F);
    normalize3(wi);
    for (int k = 0; k < 3; ++k) wi_out[k] = wi[k];
    *F_out = F;
    *side_out = side;
}

/* ---------------------------------------------------------------------------------------------- */
/* Path loop                                              */
/* ---------------------------------------------------------------------------------------------- */
typedef struct {
    const orc_scene* sc;
    const nif64* nif;        /* SIREN HDR-NIF, or NULL */
    const fr_net* fr;        /* the paper's NIF family, or NULL; both NULL -> constant env */
    int fr_fp8;              /* fr evaluated in the fp8 model (reading R24; weights already rounded) */
    double env[3];
    int32_t W, H, max_depth;
    uint64_t seed;
    cam32 cam;
} render_ctx;

typedef struct { int64_t segments, escaped, emitted, capped, rr_killed; } path_stats;

#define RR_START 3
#define MAX_TRACE 64

/* Russian roulette "with probability proportional to their radiometric throughput", from depth 3
   (PAPER.md:78, 150): survive with q = min(1, max_c beta_c) (reading R8), then beta /= q.
   Returns 0 when the path is terminated. */
static int roulette(double beta[3], int depth, double xi3) {
    if (depth < RR_START) return 1;
    double q = beta[0];
    if (beta[1] > q) q = beta[1];
    if (beta[2] > q) q = beta[2];
    if (q > 1.0) q = 1.0;
    if (xi3 >= q) return 0;
    for (int k = 0; k < 3; ++k) beta[k] /= q;
    return 1;
}

EXPORT int orc_roulette(double* beta, int32_t depth, double xi3) { return roulette(beta, depth, xi3); }

/* trace record (optional): per segment prim id (-1 miss) */
/* Optional per-segment record of one path (first-divergence classifier, tests only): segment k (0-based)
   = the k+1-th traced ray: the ray (o, d) and its hit primitive (-1 = escape) and t, the hit's edge measure
   (min barycentric, or the sphere graze measure), the signed decision deltas xi2 - F of a dielectric's
   Fresnel choice (< 0: reflect) and xi3 - q of the roulette after it (>= 0: the path ends) (+inf where no
   such decision), and the escape direction's equirect (u, v). */
typedef struct {
    int64_t* prim;      /* [max_depth] */
    double* edge;       /* [max_depth] */
    double* fres_delta;
    double* rr_delta;
    double* ray;        /* [max_depth][7]: o, d, t */
    double* uv;         /* [2] of the escape segment (-1 if none) */
    int32_t len;
} path_rec;

static void trace_path(const render_ctx* c, int64_t p, int32_t s, double L[3], path_stats* st,
                       int64_t* trace_prims, int32_t* trace_len, path_rec* rec) {
    const orc_scene* sc = c->sc;
    double xi[4];
    draw4(c->seed, (uint32_t)p, (uint32_t)s, 0u, xi);
    float d32[3];
    cam_dir32(&c->cam, c->W, c->H, (int32_t)(p % c->W), (int32_t)(p / c->W), (float)xi[0], (float)xi[1], d32);
    double o[3] = {c->cam.eye[0], c->cam.eye[1], c->cam.eye[2]};
    double d[3] = {d32[0], d32[1], d32[2]};
    double beta[3] = {1.0, 1.0, 1.0};
    L[0] = L[1] = L[2] = 0.0;
    int depth = 0;
    if (trace_len) *trace_len = 0;
    for (;;) {
        ray_pre r;
        ray_prepare(o, d, &r);
        hit_rec h;
        closest_bvh(sc, &r, &h);
        depth += 1;
        st->segments++;
        if (trace_prims && depth <= MAX_TRACE) { trace_prims[depth - 1] = h.prim; *trace_len = depth; }
        if (rec) {
            rec->prim[depth - 1] = h.prim;
            rec->edge[depth - 1] = h.prim >= 0 ? h.edge : INFINITY;
            rec->fres_delta[depth - 1] = INFINITY;
            rec->rr_delta[depth - 1] = INFINITY;
            double* ry = rec->ray + 7 * (depth - 1);
            for (int k = 0; k < 3; ++k) { ry[k] = o[k]; ry[3 + k] = d[k]; }
            ry[6] = h.prim >= 0 ? h.t : INFINITY;
            rec->len = depth;
        }
        if (h.prim < 0) {                                   /* escaped: environment light */
            double env[3];
            if (c->nif || c->fr) {
                double u, v, y[3];
                equirect(d, &u, &v);
                if (c->nif) nif_eval(c->nif, u, v, y);
                else if (c->fr_fp8) fr_net_eval_fp8(c->fr, u, v, y);
                else fr_net_eval(c->fr, u, v, y);
                for (int k = 0; k < 3; ++k) env[k] = exp(y[k]);
            } else {
                for (int k = 0; k < 3; ++k) env[k] = c->env[k];
            }
            for (int k = 0; k < 3; ++k) L[k] += beta[k] * env[k];
            st->escaped++;
            if (rec) equirect(d, &rec->uv[0], &rec->uv[1]);
            return;
        }
        uint32_t mi;
        double P[3], ng[3];
        for (int k = 0; k < 3; ++k) P[k] = o[k] + h.t * d[k];
        if (h.prim < sc->n_tris) {
            const double* v = sc->tv + 9 * h.prim;
            double e1[3] = {v[3] - v[0], v[4] - v[1], v[5] - v[2]};
            double e2[3] = {v[6] - v[0], v[7] - v[1], v[8] - v[2]};
            ng[0] = e1[1] * e2[2] - e1[2] * e2[1];
            ng[1] = e1[2] * e2[0] - e1[0] * e2[2];
            ng[2] = e1[0] * e2[1] - e1[1] * e2[0];
            normalize3(ng);
            mi = sc->tmat[h.prim];
        } else {
            const double* s4 = sc->sp + 4 * (h.prim - sc->n_tris);
            for (int k = 0; k < 3; ++k) ng[k] = (P[k] - s4[k]) / s4[3];
            mi = sc->smat[h.prim - sc->n_tris];
        }
        const in_mat* m = &sc->mats[mi];
        double cosd = dot3(d, ng);
        if (m->kind == K_EMISSIVE) {                        /* one-sided emitter, no scattering */
            if (cosd < 0.0) for (int k = 0; k < 3; ++k) L[k] += beta[k] * (double)m->emission[k];
            st->emitted++;
            return;
        }
        if (depth == c->max_depth) { st->capped++; return; }  /* depth cap: no env (reading R7) */
        draw4(c->seed, (uint32_t)p, (uint32_t)s, (uint32_t)depth, xi);
        int entering = cosd < 0.0;
        double n[3];
        for (int k = 0; k < 3; ++k) n[k] = entering ? ng[k] : -ng[k];
        double wi[3];
        int side = 1;
        if (m->kind == K_LAMBERT) {
            scatter_lambert(n, xi[0], xi[1], wi);
            for (int k = 0; k < 3; ++k) beta[k] *= (double)m->albedo[k];
        } else if (m->kind == K_MIRROR) {
            scatter_mirror(d, n, wi);
            for (int k = 0; k < 3; ++k) beta[k] *= (double)m->albedo[k];
        } else {
            double F;
            side = scatter_dielectric(d, n, entering, (double)m->ior, xi[2], wi, &F);
            if (rec) rec->fres_delta[depth - 1] = xi[2] - F;
        }
        normalize3(wi);
        /* spawn: offset along the side wi leaves to (reading R10) */
        double pm = 1.0;
        for (int k = 0; k < 3; ++k) if (fabs(P[k]) > pm) pm = fabs(P[k]);
        double eps = 1e-4 * pm;
        for (int k = 0; k < 3; ++k) { o[k] = P[k] + eps * (double)side * n[k]; d[k] = wi[k]; }
        if (rec && depth >= RR_START) {
            double q = beta[0];
            if (beta[1] > q) q = beta[1];
            if (beta[2] > q) q = beta[2];
            if (q > 1.0) q = 1.0;
            rec->rr_delta[depth - 1] = xi[3] - q;
        }
        if (!roulette(beta, depth, xi[3])) { st->rr_killed++; return; }
    }
}

typedef struct {
    const render_ctx* c;
    const int64_t* pix;
    int64_t n_pix;
    int32_t s0, s1;
    double* out;
    int tid, nthreads;
    path_stats st;
} worker_arg;

static void* worker(void* vp) {
    worker_arg* a = (worker_arg*)vp;
    memset(&a->st, 0, sizeof(a->st));
    for (int64_t i = a->tid; i < a->n_pix; i += a->nthreads) {
        double acc[3] = {0, 0, 0};
        for (int32_t s = a->s0; s < a->s1; ++s) {
            double L[3];
            trace_path(a->c, a->pix[i], s, L, &a->st, NULL, NULL, NULL);
            for (int k = 0; k < 3; ++k) acc[k] += L[k];
        }
        for (int k = 0; k < 3; ++k) a->out[3 * i + k] = acc[k];
    }
    return NULL;
}

/* Sum over samples [s0, s1) of the radiance of each listed pixel (out[3*i..] = sum, not mean).
   stats[0..4] = segments, escaped, emitted, capped, rr_killed. */
static void render_pixels(render_ctx* cp, const int64_t* pix, int64_t n_pix, int32_t s0, int32_t s1,
                          int32_t nthreads, double* out, int64_t* stats) {
    render_ctx c = *cp;
    if (nthreads < 1) nthreads = 1;
    pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * nthreads);
    worker_arg* args = (worker_arg*)malloc(sizeof(worker_arg) * nthreads);
    for (int t = 0; t < nthreads; ++t) {
        args[t] = (worker_arg){&c, pix, n_pix, s0, s1, out, t, nthreads, {0, 0, 0, 0, 0}};
        pthread_create(&th[t], NULL, worker, &args[t]);
    }
    path_stats tot = {0, 0, 0, 0, 0};
    for (int t = 0; t < nthreads; ++t) {
        pthread_join(th[t], NULL);
        tot.segments += args[t].st.segments; tot.escaped += args[t].st.escaped;
        tot.emitted += args[t].st.emitted; tot.capped += args[t].st.capped; tot.rr_killed += args[t].st.rr_killed;
    }
    if (stats) { stats[0] = tot.segments; stats[1] = tot.escaped; stats[2] = tot.emitted; stats[3] = tot.capped; stats[4] = tot.rr_killed; }
    free(th); free(args);
}

EXPORT int orc_render(const orc_scene* sc, const uint16_t* nif_blob, const double* env_rgb, int32_t W, int32_t H,
                      int32_t max_depth, uint64_t seed, const int64_t* pix, int64_t n_pix, int32_t s0, int32_t s1,
                      int32_t nthreads, double* out, int64_t* stats) {
    render_ctx c;
    c.sc = sc; c.W = W; c.H = H; c.max_depth = max_depth; c.seed = seed;
    cam_setup(&sc->cam, W, H, &c.cam);
    nif64 net;
    if (nif_blob) { nif_unpack(nif_blob, &net); c.nif = &net; }
    else c.nif = NULL;
    c.fr = NULL;
    c.fr_fp8 = 0;
    for (int k = 0; k < 3; ++k) c.env[k] = env_rgb ? env_rgb[k] : 1.0;
    render_pixels(&c, pix, n_pix, s0, s1, nthreads, out, stats);
    if (nif_blob) nif_free(&net);
    return 0;
}

/* As orc_render, with the environment given by the paper's NIF family (fr_H, fr_L; (128, 4) is the
   PT_NIF_FOURIER_RELU network); fp8 != 0 evaluates it in the fp8 model (reading R24). */
EXPORT int orc_render_fr_ex(const orc_scene* sc, int32_t fr_H, int32_t fr_L, const uint16_t* fr_blob, int32_t fp8,
                            int32_t W, int32_t H, int32_t max_depth, uint64_t seed, const int64_t* pix, int64_t n_pix,
                            int32_t s0, int32_t s1, int32_t nthreads, double* out, int64_t* stats) {
    render_ctx c;
    c.sc = sc; c.W = W; c.H = H; c.max_depth = max_depth; c.seed = seed;
    cam_setup(&sc->cam, W, H, &c.cam);
    fr_net net;
    fr_unpack(fr_H, fr_L, fr_blob, &net);
    if (fp8) fr_quantize_fp8(&net);
    c.nif = NULL;
    c.fr = &net;
    c.fr_fp8 = fp8 != 0;
    for (int k = 0; k < 3; ++k) c.env[k] = 1.0;
    render_pixels(&c, pix, n_pix, s0, s1, nthreads, out, stats);
    fr_net_free(&net);
    return 0;
}
EXPORT int orc_render_fr(const orc_scene* sc, int32_t fr_H, int32_t fr_L, const uint16_t* fr_blob, int32_t W,
                         int32_t H, int32_t max_depth, uint64_t seed, const int64_t* pix, int64_t n_pix, int32_t s0,
                         int32_t s1, int32_t nthreads, double* out, int64_t* stats) {
    return orc_render_fr_ex(sc, fr_H, fr_L, fr_blob, 0, W, H, max_depth, seed, pix, n_pix, s0, s1, nthreads, out,
                            stats);
}

/* Single path with its per-segment primitive ids (first-divergence classifier, tests only). */
EXPORT int32_t orc_trace_one(const orc_scene* sc, const uint16_t* nif_blob, const double* env_rgb, int32_t W, int32_t H,
                             int32_t max_depth, uint64_t seed, int64_t p, int32_t s, double* L, int64_t* prims) {
    render_ctx c;
    c.sc = sc; c.W = W; c.H = H; c.max_depth = max_depth; c.seed = seed;
    cam_setup(&sc->cam, W, H, &c.cam);
    nif64 net;
    if (nif_blob) { nif_unpack(nif_blob, &net); c.nif = &net; } else c.nif = NULL;
    c.fr = NULL;
    c.fr_fp8 = 0;
    for (int k = 0; k < 3; ++k) c.env[k] = env_rgb ? env_rgb[k] : 1.0;
    path_stats st = {0, 0, 0, 0, 0};
    int32_t len = 0;
    trace_path(&c, p, s, L, &st, prims, &len, NULL);
    if (nif_blob) nif_free(&net);
    return len;
}

/* Primary hits of sample `sample` for listed pixels: the fp32 camera ray widened to fp64, then the
   fp64 closest hit. edge = min barycentric (triangles) or graze measure (spheres). */
EXPORT void orc_primary(const orc_scene* sc, int32_t W, int32_t H, uint64_t seed, int32_t sample,
                        const int64_t* pix, int64_t n, int64_t* prim, double* t, double* edge) {
    cam32 k;
    cam_setup(&sc->cam, W, H, &k);
    for (int64_t i = 0; i < n; ++i) {
        double xi[4];
        int64_t p = pix[i];
        draw4(seed, (uint32_t)p, (uint32_t)sample, 0u, xi);
        float d32[3];
        cam_dir32(&k, W, H, (int32_t)(p % W), (int32_t)(p / W), (float)xi[0], (float)xi[1], d32);
        double o[3] = {k.eye[0], k.eye[1], k.eye[2]}, d[3] = {d32[0], d32[1], d32[2]};
        ray_pre r;
        ray_prepare(o, d, &r);
        hit_rec h;
        closest_bvh(sc, &r, &h);
        prim[i] = h.prim;
        t[i] = h.prim >= 0 ? h.t : INFINITY;
        edge[i] = h.prim >= 0 ? h.edge : 0.0;
    }
}

/* Table-3 AOVs of the primary hits (Sec. 4.2: normals and primary hit points): for
   listed pixels of sample `sample`, the fp64 closest hit of the fp32 camera ray (widened), the hit point
   P = o + t d, the geometric normal n_g (triangle: normalize((v1 - v0) x (v2 - v0)); sphere: (P - c) / r,
   SURVEY 8c step 6) and the barycentrics (b1, b2) = (V, W) / det of the watertight test (0 for spheres
   and misses). pos/nrm: [n][3], bary2: [n][2]; misses give prim -1 and zeros. */
EXPORT void orc_primary_aov(const orc_scene* sc, int32_t W, int32_t H, uint64_t seed, int32_t sample,
                            const int64_t* pix, int64_t n, int64_t* prim, double* t, double* pos, double* nrm,
                            double* bary2) {
    cam32 k;
    cam_setup(&sc->cam, W, H, &k);
    for (int64_t i = 0; i < n; ++i) {
        double xi[4];
        int64_t p = pix[i];
        draw4(seed, (uint32_t)p, (uint32_t)sample, 0u, xi);
        float d32[3];
        cam_dir32(&k, W, H, (int32_t)(p % W), (int32_t)(p / W), (float)xi[0], (float)xi[1], d32);
        double o[3] = {k.eye[0], k.eye[1], k.eye[2]}, d[3] = {d32[0], d32[1], d32[2]};
        ray_pre r;
        ray_prepare(o, d, &r);
        hit_rec h;
        closest_bvh(sc, &r, &h);
        prim[i] = h.prim;
        t[i] = h.prim >= 0 ? h.t : INFINITY;
        for (int a = 0; a < 3; ++a) { pos[3 * i + a] = 0.0; nrm[3 * i + a] = 0.0; }
        bary2[2 * i] = bary2[2 * i + 1] = 0.0;
        if (h.prim < 0) continue;
        double P[3];
        for (int a = 0; a < 3; ++a) P[a] = o[a] + h.t * d[a];
        double ng[3];
        if (h.prim < sc->n_tris) {
            const double* v = sc->tv + 9 * h.prim;
            double e1[3], e2[3];
            for (int a = 0; a < 3; ++a) { e1[a] = v[3 + a] - v[a]; e2[a] = v[6 + a] - v[a]; }
            ng[0] = e1[1] * e2[2] - e1[2] * e2[1];
            ng[1] = e1[2] * e2[0] - e1[0] * e2[2];
            ng[2] = e1[0] * e2[1] - e1[1] * e2[0];
            double l = sqrt(ng[0] * ng[0] + ng[1] * ng[1] + ng[2] * ng[2]);
            for (int a = 0; a < 3; ++a) ng[a] /= l;
            bary2[2 * i] = h.bary[1];
            bary2[2 * i + 1] = h.bary[2];
        } else {
            const double* s = sc->sp + 4 * (h.prim - sc->n_tris);
            for (int a = 0; a < 3; ++a) ng[a] = (P[a] - s[a]) / s[3];
        }
        for (int a = 0; a < 3; ++a) { pos[3 * i + a] = P[a]; nrm[3 * i + a] = ng[a]; }
    }
}

/* Per-segment records of the paths (listed pixels x samples [s0, s1)) for the first-divergence classifier
   (tests only): path i = pixel pix[i / ns] sample s0 + i % ns, arrays [n_paths][max_depth] (prim -2 past
   the end), ray [n_paths][max_depth][7], uv [n_paths][2] (-1 without escape), L [n_paths][3], len [n_paths]. */
EXPORT void orc_trace_paths(const orc_scene* sc, const uint16_t* nif_blob, const double* env_rgb, int32_t W, int32_t H,
                            int32_t max_depth, uint64_t seed, const int64_t* pix, int64_t n_pix, int32_t s0, int32_t s1,
                            int64_t* prim, double* edge, double* fres_delta, double* rr_delta, double* ray, double* uv,
                            double* L, int32_t* len) {
    render_ctx c;
    c.sc = sc; c.W = W; c.H = H; c.max_depth = max_depth; c.seed = seed;
    cam_setup(&sc->cam, W, H, &c.cam);
    nif64 net;
    if (nif_blob) { nif_unpack(nif_blob, &net); c.nif = &net; } else c.nif = NULL;
    c.fr = NULL;
    c.fr_fp8 = 0;
    for (int k = 0; k < 3; ++k) c.env[k] = env_rgb ? env_rgb[k] : 1.0;
    const int32_t ns = s1 - s0;
    path_stats st = {0, 0, 0, 0, 0};
    for (int64_t i = 0; i < n_pix * ns; ++i) {
        const int64_t o = i * max_depth;
        for (int32_t k = 0; k < max_depth; ++k) {
            prim[o + k] = -2; edge[o + k] = INFINITY; fres_delta[o + k] = INFINITY; rr_delta[o + k] = INFINITY;
            for (int a = 0; a < 7; ++a) ray[7 * (o + k) + a] = 0.0;
        }
        path_rec r = {prim + o, edge + o, fres_delta + o, rr_delta + o, ray + 7 * o, uv + 2 * i, 0};
        uv[2 * i] = uv[2 * i + 1] = -1.0;
        trace_path(&c, pix[i / ns], s0 + (int32_t)(i % ns), L + 3 * i, &st, NULL, NULL, &r);
        len[i] = r.len;
    }
    if (nif_blob) nif_free(&net);
}
