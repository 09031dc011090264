/*
 * bt_port.c -- C restatement of the reference hot path (TEST INFRASTRUCTURE,
 * see bt_port.h).  Reference paths are relative to /root/reference/proj.
 * Arithmetic is IEEE binary32 one operation at a time in the reference's
 * order (build with -ffp-contract=off); quadric analysis is fp64 with libm.
 */
#define _GNU_SOURCE
#include "bt_port.h"

#include <math.h>
#include <pthread.h>
#include <stdatomic.h>
#include <stdlib.h>
#include <string.h>

#define SENT 0x7FFFFFu
#define STACK_CAP 22u
#define CACHE_FLOATS 768u

typedef struct { float x, y, z; } v3;
typedef struct { float w, x, y, z; } q4;

/* ---------------------------------------------------------------- math.hpp:16-67 */
static inline v3 V(float x, float y, float z) { v3 r = {x, y, z}; return r; }
static inline v3 add(v3 a, v3 b) { return V(a.x + b.x, a.y + b.y, a.z + b.z); }
static inline v3 sub(v3 a, v3 b) { return V(a.x - b.x, a.y - b.y, a.z - b.z); }
static inline v3 mul(v3 a, float s) { return V(a.x * s, a.y * s, a.z * s); }
static inline v3 dvs(v3 a, float s) { return V(a.x / s, a.y / s, a.z / s); }
static inline float dot(v3 a, v3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
static inline v3 cross(v3 a, v3 b) { return V(a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x); }
static inline float len(v3 a) { return sqrtf(dot(a, a)); }
static inline v3 nrm(v3 a) { float l = len(a); return l > 0.0f ? dvs(a, l) : V(0, 0, 0); }
static inline float fmn(float a, float b) { return (b < a) ? b : a; } /* std::min */
static inline float fmx(float a, float b) { return (a < b) ? b : a; } /* std::max */
static inline q4 conj4(q4 q) { q4 r = {q.w, -q.x, -q.y, -q.z}; return r; }
static inline v3 rot(q4 q, v3 v) {
    v3 u = V(q.x, q.y, q.z);
    v3 t = mul(cross(u, v), 2.0f);
    return add(add(v, mul(t, q.w)), cross(u, t));
}

/* ---------------------------------------------------------------- blob (linear_tree.cpp:9-36) */
static inline uint32_t blob(const float* data, uint32_t w) { uint32_t b; memcpy(&b, &data[4 * w], 4); return b; }
static inline int b_prim(uint32_t b) { return (int)(b >> 31); }
static inline uint32_t b_op(uint32_t b) { return (b >> 26) & 31u; }
static inline uint32_t b_ign(uint32_t b) { return (b >> 24) & 3u; }
static inline int b_left(uint32_t b) { return (int)((b >> 23) & 1u); }
static inline uint32_t b_anc(uint32_t b) { return b & SENT; }
static inline uint32_t b_set_anc(uint32_t b, uint32_t a) { return (b & ~SENT) | a; }
static inline const float* params_at(const float* data, uint32_t w) { return data + 4 * (w + 1); }

static uint32_t shape_count(uint32_t kind) {
    static const uint32_t n[6] = {1, 3, 2, 3, 3, 10};
    return kind < 6 ? n[kind] : 0;
}

/* ---------------------------------------------------------------- field.cpp:221-284 */
static float prim_eval(uint32_t kind, const float* P, v3 p) {
    v3 t = V(P[0], P[1], P[2]);
    q4 q = {P[3], P[4], P[5], P[6]};
    v3 l = rot(conj4(q), sub(p, t));
    const float* s = P + 7;
    float v = 0.0f;
    if (kind == 0) {
        v = len(l) - s[0];
    } else if (kind == 1) {
        float k0 = len(V(l.x / s[0], l.y / s[1], l.z / s[2]));
        float k1 = len(V(l.x / (s[0] * s[0]), l.y / (s[1] * s[1]), l.z / (s[2] * s[2])));
        v = (k1 <= 0.0f) ? -fmn(s[0], fmn(s[1], s[2])) : k0 * (k0 - 1.0f) / k1;
    } else if (kind == 2) {
        float qx = sqrtf(l.x * l.x + l.z * l.z) - s[0];
        v = sqrtf(qx * qx + l.y * l.y) - s[1];
    } else if (kind == 3) {
        v3 q = V(fabsf(l.x) - s[0], fabsf(l.y) - s[1], fabsf(l.z) - s[2]);
        v3 o = V(fmx(q.x, 0.0f), fmx(q.y, 0.0f), fmx(q.z, 0.0f));
        v = len(o) + fmn(fmx(q.x, fmx(q.y, q.z)), 0.0f);
    } else if (kind == 4) {
        float qx = sqrtf(l.x * l.x + l.z * l.z), qy = l.y;
        float b = (s[0] - s[1]) / s[2];
        float a = sqrtf(1.0f - b * b);
        float k = qx * (-b) + qy * a;
        if (k < 0.0f) v = sqrtf(qx * qx + qy * qy) - s[0];
        else if (k > a * s[2]) { float dy = qy - s[2]; v = sqrtf(qx * qx + dy * dy) - s[1]; }
        else v = qx * a + qy * b - s[0];
    } else if (kind == 5) {
        const float* c = s;
        float gx = 2.0f * (c[0] * l.x) + c[3] * l.y + c[4] * l.z + c[6];
        float gy = 2.0f * (c[1] * l.y) + c[3] * l.x + c[5] * l.z + c[7];
        float gz = 2.0f * (c[2] * l.z) + c[4] * l.x + c[5] * l.y + c[8];
        float f0 = c[0] * l.x * l.x + c[1] * l.y * l.y + c[2] * l.z * l.z + c[3] * l.x * l.y + c[4] * l.x * l.z +
                   c[5] * l.y * l.z + c[6] * l.x + c[7] * l.y + c[8] * l.z + c[9];
        float g = sqrtf(gx * gx + gy * gy + gz * gz);
        v = f0 / fmx(g, 1e-4f);
    }
    return isnan(v) ? 0.0f : v;
}

/* ---------------------------------------------------------------- field.cpp:399-454 */
static float csg(uint32_t fl, float a, float b) { return fl == 0 ? fmn(a, b) : fl == 1 ? fmx(a, b) : fmx(a, -b); }
static float disp(float a, float b, float k) {
    if (!(k > 0.0f)) return 0.0f;
    float ad = fabsf(a - b);
    if (!(ad < k)) return 0.0f;
    float t = 1.0f - ad / k;
    return (k / 6.0f) * t * t * t;
}
static float smooth(uint32_t fl, float a, float b, float k) {
    float v = fl == 0 ? fmn(a, b) - disp(a, b, k) : fl == 1 ? fmx(a, b) + disp(a, b, k) : fmx(a, -b) + disp(a, -b, k);
    return isnan(v) ? 0.0f : v;
}
static float brange(float x, float k, float d) {
    float v = k * fmx(1.0f - 6.0f * x / (6.0f * d - k), 0.0f);
    return isnan(v) ? 0.0f : v;
}
static float op_eval(uint32_t code, const float* P, float a, float b) {
    if (code == 0) return INFINITY;
    if (code == 1) return b;
    if (code == 2) return a;
    uint32_t fl = (code - 3) % 3;
    if (code <= 5) return csg(fl, a, b);
    if (code <= 8) return smooth(fl, a, b, P[0]);
    float k = P[0], d = P[1];
    if (a > d || b > d) return csg(fl, a, b);
    float g = smooth(fl, a, b, k);
    float kp = fl == 0 ? brange(g, k, d) : fl == 1 ? fmn(brange(g, k, d), k) : fmn(brange(fabsf(g), k, d), k);
    return smooth(fl, a, b, kp);
}

float port_eval_primitive(uint32_t kind, const float* params, float x, float y, float z) {
    return prim_eval(kind, params, V(x, y, z));
}
float port_eval_operator(uint32_t code, const float* params, float f0, float f1) {
    return op_eval(code, params, f0, f1);
}

/* eval_full (traversal.cpp:126-141), heap stack sized to the tree */
float port_eval_full(const port_tree* t, float x, float y, float z) {
    float* st = (float*)malloc(sizeof(float) * (t->nnodes + 1));
    uint32_t sp = 0;
    v3 p = V(x, y, z);
    for (uint32_t i = 0; i < t->nnodes; ++i) {
        const bt_node* n = &t->nodes[i];
        const float* P = params_at(t->data, n->word);
        if (n->isPrimitive) {
            st[sp++] = prim_eval(n->nodeOp, P, p);
        } else {
            float r = st[--sp];
            float l = st[--sp];
            st[sp++] = op_eval(n->nodeOp, P, l, r);
        }
    }
    float v = st[0];
    free(st);
    return v;
}

/* ---------------------------------------------------------------- (a) linear_tree.cpp:170-283 */
void port_roi(const port_tree* t, float* out) {
    for (uint32_t i = 0; i < t->nnodes; ++i) out[i] = 0.0f;
    for (uint32_t i = t->nnodes; i-- > 0;) {
        const bt_node* n = &t->nodes[i];
        if (n->isPrimitive) continue;
        float u = out[i];
        if (n->nodeOp >= 9 && n->nodeOp <= 11) u = fmx(u, params_at(t->data, n->word)[1]);
        out[n->leftChild] = u;
        out[n->rightChild] = u;
    }
}

static void sort3(double* v) {
    double t;
    if (v[1] < v[0]) { t = v[0]; v[0] = v[1]; v[1] = t; }
    if (v[2] < v[1]) { t = v[1]; v[1] = v[2]; v[2] = t; }
    if (v[1] < v[0]) { t = v[0]; v[0] = v[1]; v[1] = t; }
}

/* analyze_quadric (field.cpp:110-172) */
static void quadric_info(const float* c, v3* center, float* iso, float* lmin, float* lmax) {
    double a11 = c[0], a22 = c[1], a33 = c[2], a12 = c[3], a13 = c[4], a23 = c[5];
    double bx = c[6], by = c[7], bz = c[8], cc = c[9], e[3];
    double p1 = a12 * a12 + a13 * a13 + a23 * a23;
    if (p1 == 0.0) {
        e[0] = a11; e[1] = a22; e[2] = a33;
    } else {
        double q = (a11 + a22 + a33) / 3.0;
        double p2 = (a11 - q) * (a11 - q) + (a22 - q) * (a22 - q) + (a33 - q) * (a33 - q) + 2.0 * p1;
        double p = sqrt(p2 / 6.0);
        double b11 = (a11 - q) / p, b22 = (a22 - q) / p, b33 = (a33 - q) / p, b12 = a12 / p, b13 = a13 / p,
               b23 = a23 / p;
        double det = b11 * (b22 * b33 - b23 * b23) - b12 * (b12 * b33 - b23 * b13) + b13 * (b12 * b23 - b22 * b13);
        double r = det / 2.0;
        r = r < -1.0 ? -1.0 : (1.0 < r ? 1.0 : r);
        double phi = acos(r) / 3.0;
        double e1 = q + 2.0 * p * cos(phi);
        double e3 = q + 2.0 * p * cos(phi + 2.0 * M_PI / 3.0);
        e[0] = e3; e[1] = 3.0 * q - e1 - e3; e[2] = e1;
    }
    sort3(e);
    *lmin = (float)e[0];
    *lmax = (float)e[2];
    *center = V(0, 0, 0);
    *iso = 0.0f;
    if (!(e[0] > 0.0)) return;
    double det = a11 * (a22 * a33 - a23 * a23) - a12 * (a12 * a33 - a23 * a13) + a13 * (a12 * a23 - a22 * a13);
    double rx = -bx / 2.0, ry = -by / 2.0, rz = -bz / 2.0;
    double mx = (rx * (a22 * a33 - a23 * a23) - a12 * (ry * a33 - a23 * rz) + a13 * (ry * a23 - a22 * rz)) / det;
    double my = (a11 * (ry * a33 - a23 * rz) - rx * (a12 * a33 - a23 * a13) + a13 * (a12 * rz - ry * a13)) / det;
    double mz = (a11 * (a22 * rz - ry * a23) - a12 * (a12 * rz - ry * a13) + rx * (a12 * a23 - a22 * a13)) / det;
    *center = V((float)mx, (float)my, (float)mz);
    double mAm = mx * (a11 * mx + a12 * my + a13 * mz) + my * (a12 * mx + a22 * my + a23 * mz) +
                 mz * (a13 * mx + a23 * my + a33 * mz);
    *iso = (float)(mAm - cc);
}

void port_vois(const port_tree* t, const float* roi, float margin, bt_voi* out) {
    uint32_t ord = 0;
    for (uint32_t i = 0; i < t->nprims; ++i) {
        uint32_t w = t->prims[i];
        while (t->nodes[ord].word != w) ++ord; /* both ascending */
        float u = roi[ord] + margin + 1e-5f;
        const float* P = params_at(t->data, w);
        const float* s = P + 7;
        v3 tr = V(P[0], P[1], P[2]);
        q4 q = {P[3], P[4], P[5], P[6]};
        bt_voi* v = &out[i];
        memset(v, 0, sizeof(*v));
        v->rotation[0] = 1.0f;
        v->primitiveWord = w;
        v->center[0] = tr.x; v->center[1] = tr.y; v->center[2] = tr.z;
        switch (b_op(blob(t->data, w))) {
            case 0: v->radius = s[0] + u; break;
            case 1: {
                float rmin = fmn(s[0], fmn(s[1], s[2])), rmax = fmx(s[0], fmx(s[1], s[2]));
                float d = u * (rmax / rmin);
                v->family = 1;
                v->rotation[0] = q.w; v->rotation[1] = q.x; v->rotation[2] = q.y; v->rotation[3] = q.z;
                v->halfExtents[0] = s[0] + d; v->halfExtents[1] = s[1] + d; v->halfExtents[2] = s[2] + d;
                break;
            }
            case 2: v->radius = s[0] + s[1] + u; break;
            case 3:
                v->family = 1;
                v->rotation[0] = q.w; v->rotation[1] = q.x; v->rotation[2] = q.y; v->rotation[3] = q.z;
                v->halfExtents[0] = s[0] + u; v->halfExtents[1] = s[1] + u; v->halfExtents[2] = s[2] + u;
                break;
            case 4: {
                v3 e = add(tr, rot(q, V(0, s[2], 0)));
                v->family = 2;
                v->axisEnd[0] = e.x; v->axisEnd[1] = e.y; v->axisEnd[2] = e.z;
                v->radius = fmx(s[0], s[1]) + u;
                break;
            }
            case 5: {
                v3 qc; float iso, lmin, lmax;
                quadric_info(s, &qc, &iso, &lmin, &lmax);
                v3 c = add(tr, rot(q, qc));
                v->center[0] = c.x; v->center[1] = c.y; v->center[2] = c.z;
                float r0 = sqrtf(fmx(iso, 0.0f) / lmin);
                v->radius = r0 + 2.0f * u * (lmax / lmin);
                break;
            }
        }
    }
}

/* ---------------------------------------------------------------- camera.cpp:29-37 */
typedef struct { v3 o, d; float ddf; } ray_t;
static ray_t ray_at(const bt_camera* c, float px, float py) {
    v3 f = V(c->forward[0], c->forward[1], c->forward[2]);
    v3 r = V(c->right[0], c->right[1], c->right[2]);
    v3 u = V(c->up[0], c->up[1], c->up[2]);
    float sx = (2.0f * px / (float)c->width - 1.0f) * c->tanHalf * c->aspect;
    float sy = (1.0f - 2.0f * py / (float)c->height) * c->tanHalf;
    ray_t R;
    R.o = V(c->position[0], c->position[1], c->position[2]);
    R.d = nrm(add(add(f, mul(r, sx)), mul(u, sy)));
    R.ddf = dot(R.d, f);
    return R;
}
static ray_t pixel_ray(const bt_camera* c, int x, int y) { return ray_at(c, (float)x + 0.5f, (float)y + 0.5f); }
static float ndc(const bt_camera* c, float vz) { return (c->invNear - 1.0f / vz) * c->invDepthRange; }
static float vz_of_ndc(const bt_camera* c, float z) { return 1.0f / (c->invNear - z / c->invDepthRange); }

/* ---------------------------------------------------------------- (b) abuffer.cpp:18-225 */
static int isect_sphere(v3 o, v3 d, v3 c, float r, float* t0, float* t1) {
    v3 oc = sub(o, c);
    float b = dot(oc, d);
    float cc = dot(oc, oc) - r * r;
    float disc = b * b - cc;
    if (disc < 0.0f) return 0;
    float s = sqrtf(disc);
    *t0 = -b - s;
    *t1 = -b + s;
    return 1;
}

static int isect_volume(const bt_voi* v, v3 o, v3 d, float* te, float* tx) {
    v3 c = V(v->center[0], v->center[1], v->center[2]);
    if (v->family == 0) return isect_sphere(o, d, c, v->radius, te, tx);
    if (v->family == 1) {
        q4 inv = conj4((q4){v->rotation[0], v->rotation[1], v->rotation[2], v->rotation[3]});
        v3 lo = rot(inv, sub(o, c)), ld = rot(inv, d);
        float oa[3] = {lo.x, lo.y, lo.z}, da[3] = {ld.x, ld.y, ld.z};
        float lo_t = -INFINITY, hi_t = INFINITY;
        for (int i = 0; i < 3; ++i) {
            float h = v->halfExtents[i];
            if (fabsf(da[i]) < 1e-12f) {
                if (fabsf(oa[i]) > h) return 0;
                continue;
            }
            float id = 1.0f / da[i];
            float a = (-h - oa[i]) * id, b = (h - oa[i]) * id;
            if (a > b) { float t = a; a = b; b = t; }
            lo_t = fmx(lo_t, a);
            hi_t = fmn(hi_t, b);
            if (lo_t > hi_t) return 0;
        }
        *te = lo_t;
        *tx = hi_t;
        return 1;
    }
    /* capsule */
    v3 e = V(v->axisEnd[0], v->axisEnd[1], v->axisEnd[2]);
    v3 ba = sub(e, c), oa = sub(o, c);
    float baba = dot(ba, ba), bard = dot(ba, d), baoa = dot(ba, oa), r = v->radius;
    float enter = INFINITY, exit_ = -INFINITY;
    int any = 0;
    float a = baba - bard * bard;
    if (a > 1e-12f * baba) {
        float b = baba * dot(oa, d) - baoa * bard;
        float cc = baba * dot(oa, oa) - baoa * baoa - r * r * baba;
        float disc = b * b - a * cc;
        if (disc >= 0.0f) {
            float s = sqrtf(disc);
            float ts[2] = {(-b - s) / a, (-b + s) / a};
            for (int i = 0; i < 2; ++i) {
                float y = baoa + ts[i] * bard;
                if (y >= 0.0f && y <= baba) { enter = fmn(enter, ts[i]); exit_ = fmx(exit_, ts[i]); any = 1; }
            }
        }
    }
    for (int cap = 0; cap < 2; ++cap) {
        float s0, s1;
        if (!isect_sphere(o, d, cap ? e : c, r, &s0, &s1)) continue;
        float ts[2] = {s0, s1};
        for (int i = 0; i < 2; ++i) {
            float y = baoa + ts[i] * bard;
            if ((cap == 0 && y <= 0.0f) || (cap == 1 && y >= baba)) {
                enter = fmn(enter, ts[i]); exit_ = fmx(exit_, ts[i]); any = 1;
            }
        }
    }
    if (!any) return 0;
    *te = enter;
    *tx = exit_;
    return 1;
}

typedef struct { v3 axis; float cs, sn; } cone_t;
static cone_t tile_cone(const bt_camera* c, int tx, int ty) {
    float x0 = (float)(tx * 8), y0 = (float)(ty * 8), x1 = x0 + 8, y1 = y0 + 8;
    float pxs[8] = {x0, x1, x0, x1, 0.5f * (x0 + x1), 0.5f * (x0 + x1), x0, x1};
    float pys[8] = {y0, y0, y1, y1, y0, y1, 0.5f * (y0 + y1), 0.5f * (y0 + y1)};
    v3 d[8], axis = V(0, 0, 0);
    for (int i = 0; i < 8; ++i) { d[i] = ray_at(c, pxs[i], pys[i]).d; axis = add(axis, d[i]); }
    axis = nrm(axis);
    float cs = 1.0f;
    for (int i = 0; i < 8; ++i) cs = fmn(cs, dot(axis, d[i]));
    cs = fmx(cs - 1e-3f, -1.0f);
    cone_t k = {axis, cs, sqrtf(fmx(1.0f - cs * cs, 0.0f))};
    return k;
}

typedef struct { bt_fragment* v; uint32_t n, cap; } list_t;

static void list_insert(list_t* l, bt_fragment f) {
    /* upper_bound on (zEntry, word) (abuffer.cpp:166-173) */
    uint32_t lo = 0, hi = l->n;
    while (lo < hi) {
        uint32_t mid = (lo + hi) / 2;
        const bt_fragment* m = &l->v[mid];
        int less = f.zEntry < m->zEntry || (f.zEntry == m->zEntry && f.primitiveWord < m->primitiveWord);
        if (less) hi = mid; else lo = mid + 1;
    }
    if (l->n == l->cap) {
        l->cap = l->cap ? 2 * l->cap : 8;
        l->v = (bt_fragment*)realloc(l->v, l->cap * sizeof(bt_fragment));
    }
    memmove(&l->v[lo + 1], &l->v[lo], (l->n - lo) * sizeof(bt_fragment));
    l->v[lo] = f;
    l->n++;
}

int port_rasterize(const bt_voi* vois, uint32_t n, const bt_camera* cam, uint32_t* offsets, bt_fragment* frags,
                   uint64_t cap, uint64_t* total) {
    int tx = (cam->width + 7) / 8, ty = (cam->height + 7) / 8;
    size_t T = (size_t)tx * ty;
    cone_t* cones = (cone_t*)malloc(T * sizeof(cone_t));
    list_t* lists = (list_t*)calloc(T, sizeof(list_t));
    for (int y = 0; y < ty; ++y)
        for (int x = 0; x < tx; ++x) cones[(size_t)y * tx + x] = tile_cone(cam, x, y);
    v3 apex = V(cam->position[0], cam->position[1], cam->position[2]);
    v3 fwd = V(cam->forward[0], cam->forward[1], cam->forward[2]);
    for (uint32_t i = 0; i < n; ++i) {
        const bt_voi* v = &vois[i];
        v3 bc = V(v->center[0], v->center[1], v->center[2]);
        float br = v->radius;
        if (v->family == 1) br = len(V(v->halfExtents[0], v->halfExtents[1], v->halfExtents[2]));
        if (v->family == 2) {
            v3 e = V(v->axisEnd[0], v->axisEnd[1], v->axisEnd[2]);
            bc = mul(add(bc, e), 0.5f);
            br = len(sub(e, V(v->center[0], v->center[1], v->center[2]))) * 0.5f + v->radius;
        }
        float vz = dot(sub(bc, apex), fwd);
        if (vz + br < cam->nearZ || vz - br > cam->farZ) continue;
        for (int y = 0; y < ty; ++y)
            for (int x = 0; x < tx; ++x) {
                size_t ti = (size_t)y * tx + x;
                const cone_t* k = &cones[ti];
                v3 w = sub(bc, apex);
                float xx = dot(w, k->axis);
                float yy = dot(w, w) - xx * xx;
                if (!(k->cs * sqrtf(fmx(yy, 0.0f)) - k->sn * xx <= br)) continue;
                float entry = INFINITY, ex = -INFINITY;
                int anyHit = 0;
                int xe = (x + 1) * 8 < cam->width ? (x + 1) * 8 : cam->width;
                int ye = (y + 1) * 8 < cam->height ? (y + 1) * 8 : cam->height;
                for (int py = y * 8; py < ye; ++py)
                    for (int px = x * 8; px < xe; ++px) {
                        ray_t R = pixel_ray(cam, px, py);
                        float t0, t1;
                        if (!isect_volume(v, R.o, R.d, &t0, &t1)) continue;
                        float vz0 = t0 * R.ddf, vz1 = t1 * R.ddf;
                        if (vz1 < cam->nearZ || vz0 > cam->farZ) continue;
                        vz0 = fmx(vz0, cam->nearZ);
                        vz1 = fmn(vz1, cam->farZ);
                        entry = fmn(entry, ndc(cam, vz0));
                        ex = fmx(ex, ndc(cam, vz1));
                        anyHit = 1;
                    }
                if (anyHit) {
                    bt_fragment f = {v->primitiveWord, entry, ex};
                    list_insert(&lists[ti], f);
                }
            }
    }
    uint64_t m = 0;
    int rc = 0;
    for (size_t t = 0; t < T; ++t) {
        if (offsets) offsets[t] = (uint32_t)m;
        for (uint32_t j = 0; j < lists[t].n; ++j) {
            if (frags) {
                if (m >= cap) rc = 1; else frags[m] = lists[t].v[j];
            }
            ++m;
        }
        free(lists[t].v);
    }
    if (offsets) offsets[T] = (uint32_t)m;
    if (total) *total = m;
    free(lists);
    free(cones);
    return rc;
}

/* ---------------------------------------------------------------- (c) tracer.cpp / traversal */
typedef struct { uint32_t word; float zEntry, zExit; } active_t;

typedef struct {
    const bt_fragment* list;
    uint32_t n, cursor, nact;
    active_t act[BT_MAX_OVERLAP];
    float zEnd;
} fetch_t;

/* fetch_interval (tracer.cpp:50-103); returns 0 when exhausted */
static int fetch(fetch_t* s, const bt_camera* cam, const bt_render_config* cfg, float* zb, float* ze) {
    uint32_t m = 0;
    for (uint32_t i = 0; i < s->nact; ++i)
        if (!(s->act[i].zExit <= s->zEnd)) s->act[m++] = s->act[i];
    int expired = m != s->nact;
    s->nact = m;
    int hasNext = s->cursor < s->n;
    if (s->nact == 0 && !hasNext) return 0;
    float zBegin = s->zEnd;
    if (hasNext) zBegin = fmx(s->zEnd, s->list[s->cursor].zEntry);
    float window = cfg->fetchWindow;
    if (!(window > 0.0f)) window = (cam->farZ - cam->nearZ) / 20.0f;
    float zbv = vz_of_ndc(cam, zBegin);
    float maxExit = -INFINITY;
    for (uint32_t i = 0; i < s->nact; ++i) maxExit = fmx(maxExit, s->act[i].zExit);
    uint32_t fetched = 0;
    while (s->cursor < s->n) {
        bt_fragment c = s->list[s->cursor];
        if (s->nact) {
            if (c.zEntry > maxExit || fetched >= cfg->maxNewPerFetch || s->nact >= cfg->maxOverlap ||
                vz_of_ndc(cam, c.zEntry) - zbv >= window)
                break;
        }
        uint32_t pos = 0;
        while (pos < s->nact && s->act[pos].word < c.primitiveWord) ++pos;
        memmove(&s->act[pos + 1], &s->act[pos], (s->nact - pos) * sizeof(active_t));
        s->act[pos].word = c.primitiveWord;
        s->act[pos].zEntry = c.zEntry;
        s->act[pos].zExit = c.zExit;
        s->nact++;
        maxExit = fmx(maxExit, c.zExit);
        s->cursor++;
        fetched++;
    }
    float zEnd = maxExit;
    if (s->cursor < s->n) zEnd = fmn(s->list[s->cursor].zEntry, maxExit);
    if (zEnd <= zBegin && fetched == 0 && !expired) {
        float mn = INFINITY;
        for (uint32_t i = 0; i < s->nact; ++i) mn = fmn(mn, s->act[i].zExit);
        zEnd = mn;
    }
    s->zEnd = zEnd;
    *zb = zBegin;
    *ze = zEnd;
    return 1;
}

typedef struct {
    uint32_t blob[2 * BT_MAX_OVERLAP];
    const float* params[2 * BT_MAX_OVERLAP];
    uint32_t n, prims, cacheFloats;
    int rootUsed;
} view_t;

static uint32_t nfloats(uint32_t b) {
    if (b_prim(b)) return 7 + shape_count(b_op(b));
    return (b_op(b) >= 6 && b_op(b) <= 11) ? 2 : 0;
}

/* append (traversal.cpp:41-54); returns 0 on ViewOverflow */
static int vappend(view_t* v, const float* data, uint32_t b, uint32_t w, int copy, uint32_t capacity) {
    if (v->n >= capacity) return 0;
    uint32_t f = copy ? nfloats(b) : 0;
    if (f && v->cacheFloats + f <= CACHE_FLOATS) v->cacheFloats += f;
    v->blob[v->n] = b;
    v->params[v->n] = params_at(data, w);
    v->n++;
    return 1;
}

/* build_pruned_view = sparse_traverse + ViewBuildVisitor (traversal.hpp:68-117,
 * traversal.cpp:36-99).  Returns 0 ok, 1 on stack/view overflow. */
static int build_view(const float* data, const active_t* act, uint32_t n, view_t* v) {
    v->n = v->prims = v->cacheFloats = 0;
    v->rootUsed = 0;
    if (n == 0) return 0;
    uint32_t capacity = 2 * n - 1, sp = 0;
    uint32_t sb[STACK_CAP];
    uint8_t su[STACK_CAP];
    for (uint32_t i = 0; i < n; ++i) {
        uint32_t w = act[i].word, b = blob(data, w);
        if (!vappend(v, data, b, w, 1, capacity)) return 1;
        v->prims++;
        uint8_t d = 1;
        if (sp && b_anc(sb[sp - 1]) < b_anc(b)) b = b_set_anc(b, b_anc(sb[sp - 1]));
        for (;;) {
            int shadowed = (i + 1 < n) && b_anc(b) > act[i + 1].word;
            int last = (i + 1 == n) && sp == 0 && b_anc(b) == SENT;
            if (shadowed || last) break;
            if (b_anc(b) == SENT) return 1; /* logic error: walked past the root */
            uint32_t opw = b_anc(b);
            int fromLeft = b_left(b);
            b = blob(data, opw);
            int combined = 0;
            if (sp) {
                uint32_t cb = sb[sp - 1];
                if (opw == b_anc(cb) || (b_anc(b) >= b_anc(cb) && (b_anc(b) == SENT || b_left(b)))) {
                    uint8_t ch = (uint8_t)((su[sp - 1] << 1) | d);
                    uint8_t use = ((~ch & b_ign(b)) & 3u) == 0 ? ch : 0;
                    uint32_t stored = use != 3 ? ((b & ~(31u << 26)) | ((uint32_t)use << 26)) : b;
                    if (!vappend(v, data, stored, opw, use == 3, capacity)) return 1;
                    d = use ? 1 : 0;
                    sp--;
                    combined = 1;
                }
            }
            if (!combined && (b_ign(b) & (fromLeft ? 1u : 2u))) d = 0;
            if (sp && b_anc(sb[sp - 1]) < b_anc(b)) b = b_set_anc(b, b_anc(sb[sp - 1]));
        }
        if (sp >= STACK_CAP) return 1;
        sb[sp] = b;
        su[sp] = d;
        sp++;
    }
    v->rootUsed = su[sp - 1] != 0;
    return sp == 1 ? 0 : 1;
}

/* eval_pruned (traversal.cpp:101-124); *err set on stack overflow */
static float eval_view(const view_t* v, v3 p, int* err) {
    if (!v->rootUsed) return INFINITY;
    float st[STACK_CAP];
    uint32_t sp = 0;
    for (uint32_t i = 0; i < v->n; ++i) {
        uint32_t b = v->blob[i];
        float val;
        if (b_prim(b)) {
            val = prim_eval(b_op(b), v->params[i], p);
        } else {
            float r = st[--sp];
            float l = st[--sp];
            val = op_eval(b_op(b), v->params[i], l, r);
        }
        if (sp >= STACK_CAP) { *err = 1; return 0.0f; }
        st[sp++] = val;
    }
    return st[sp - 1];
}

typedef float (*field_fn)(void* ctx, float t);

/* sphere_trace_interval (tracer.hpp:99-177) */
static int trace(field_fn F, void* ctx, float t0, float t1, const bt_render_config* cfg, uint32_t* evals,
                 float* tHit, int* err) {
    if (t0 > t1) return 0;
    float invL = 1.0f / cfg->lipschitz;
    float t = t0, f = F(ctx, t);
    ++*evals;
    if (*err) return 0;
    if (f <= cfg->hitEpsilon) { *tHit = t; return 1; }
    int relaxOn = 1, savedValid = 0;
    float savedT = 0, savedF = 0;
    for (;;) {
        float r = f * invL;
        if (!isfinite(r)) return 0;
        float step = relaxOn ? cfg->relax * r : r;
        step = fmx(step, cfg->minStep);
        float tn = t + step, fn = 0.0f;
        int reused = 0;
        if (savedValid && tn >= savedT) {
            if (savedT >= t + cfg->minStep && savedT <= t1) { tn = savedT; fn = savedF; reused = 1; }
            savedValid = 0;
            relaxOn = 1;
        }
        if (tn > t1) {
            if (t >= t1) return 0;
            tn = t1;
            reused = 0;
        }
        if (!reused) {
            fn = F(ctx, tn);
            ++*evals;
            if (*err) return 0;
        }
        int over = !reused && relaxOn && ((tn - t) * cfg->lipschitz >= f + fabsf(fn) || fn < -cfg->hitEpsilon);
        if (over) {
            savedT = tn; savedF = fn; savedValid = 1; relaxOn = 0;
            float tb = t + fmx(r, cfg->minStep);
            if (tb >= savedT) {
                t = savedT; f = savedF; savedValid = 0; relaxOn = 1;
            } else if (tb > t1) {
                return 0;
            } else {
                t = tb;
                f = F(ctx, tb);
                ++*evals;
                if (*err) return 0;
            }
            if (f <= cfg->hitEpsilon) { *tHit = t; return 1; }
            continue;
        }
        if (fn <= cfg->hitEpsilon) { *tHit = tn; return 1; }
        if (tn >= t1) return 0;
        t = tn;
        f = fn;
    }
}

typedef struct { const view_t* v; v3 o, d; int* err; } view_ctx;
static float view_field(void* c, float t) {
    view_ctx* k = (view_ctx*)c;
    return eval_view(k->v, add(k->o, mul(k->d, t)), k->err);
}

/* parallel-for over an index range with an atomic cursor (tracer.cpp:117-137) */
typedef struct { atomic_uint next; uint32_t count; void (*fn)(void*, uint32_t); void* arg; } pool_t;
static void* pool_worker(void* p) {
    pool_t* P = (pool_t*)p;
    for (;;) {
        uint32_t i = atomic_fetch_add(&P->next, 1u);
        if (i >= P->count) break;
        P->fn(P->arg, i);
    }
    return NULL;
}
static void parallel_for(uint32_t count, int threads, void (*fn)(void*, uint32_t), void* arg) {
    pool_t P;
    atomic_init(&P.next, 0u);
    P.count = count;
    P.fn = fn;
    P.arg = arg;
    if (threads <= 1) { pool_worker(&P); return; }
    pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)threads);
    for (int i = 0; i < threads - 1; ++i) pthread_create(&th[i], NULL, pool_worker, &P);
    pool_worker(&P);
    for (int i = 0; i < threads - 1; ++i) pthread_join(th[i], NULL);
    free(th);
}

typedef struct {
    const port_tree* t;
    const bt_camera* cam;
    const bt_render_config* cfg;
    const uint32_t* offsets;
    const bt_fragment* frags;
    uint8_t* hit;
    float* depth;
    uint32_t* evalCount;
    uint32_t *tmo, *tcb;
    uint8_t* terr;
    _Atomic uint64_t fe, rnv, pe;
    _Atomic uint32_t mo, mc;
} rt_args;

static void atomic_max32(_Atomic uint32_t* a, uint32_t v) {
    uint32_t cur = atomic_load(a);
    while (cur < v && !atomic_compare_exchange_weak(a, &cur, v)) {
    }
}

/* render_tiles, one tile (tracer.cpp:155-232) */
static void render_tile(void* p, uint32_t tile) {
    rt_args* A = (rt_args*)p;
    const bt_camera* cam = A->cam;
    int tilesX = (cam->width + 7) / 8;
    int tx = (int)(tile % (uint32_t)tilesX), ty = (int)(tile / (uint32_t)tilesX);
    uint32_t off = A->offsets[tile], cnt = A->offsets[tile + 1] - off;
    if (cnt == 0) return;
    ray_t rays[64];
    size_t pix[64];
    int found[64], npx = 0;
    int ye = (ty + 1) * 8 < cam->height ? (ty + 1) * 8 : cam->height;
    int xe = (tx + 1) * 8 < cam->width ? (tx + 1) * 8 : cam->width;
    for (int y = ty * 8; y < ye; ++y)
        for (int x = tx * 8; x < xe; ++x) {
            rays[npx] = pixel_ray(cam, x, y);
            pix[npx] = (size_t)y * cam->width + x;
            found[npx] = 0;
            ++npx;
        }
    fetch_t* fs = (fetch_t*)calloc(1, sizeof(fetch_t));
    view_t* view = (view_t*)malloc(sizeof(view_t));
    fs->list = A->frags + off;
    fs->n = cnt;
    uint64_t fe = 0, rnv = 0, pe = 0;
    uint32_t mo = 0, mc = 0;
    int remaining = npx, err = 0;
    while (remaining > 0) {
        float zb, ze;
        if (!fetch(fs, cam, A->cfg, &zb, &ze)) break;
        if (fs->nact > A->tmo[tile]) A->tmo[tile] = fs->nact;
        if (fs->nact > mo) mo = fs->nact;
        if (build_view(A->t->data, fs->act, fs->nact, view)) { err = 1; break; }
        if (view->cacheFloats * 4 > A->tcb[tile]) A->tcb[tile] = view->cacheFloats * 4;
        if (view->cacheFloats * 4 > mc) mc = view->cacheFloats * 4;
        if (!view->rootUsed) continue;
        if (ze <= zb) continue;
        float vz0 = vz_of_ndc(cam, zb), vz1 = vz_of_ndc(cam, ze);
        for (int i = 0; i < npx && !err; ++i) {
            if (found[i]) continue;
            uint32_t ev = 0;
            float tHit = 0.0f;
            view_ctx k = {view, rays[i].o, rays[i].d, &err};
            int h = trace(view_field, &k, vz0 / rays[i].ddf, vz1 / rays[i].ddf, A->cfg, &ev, &tHit, &err);
            if (err) break;
            A->evalCount[pix[i]] += ev;
            fe += ev;
            rnv += (uint64_t)ev * view->n;
            pe += (uint64_t)ev * view->prims;
            if (h) {
                A->hit[pix[i]] = 1;
                A->depth[pix[i]] = tHit;
                found[i] = 1;
                --remaining;
            }
        }
        if (err) break;
    }
    if (err) A->terr[tile] = 1;
    atomic_fetch_add(&A->fe, fe);
    atomic_fetch_add(&A->rnv, rnv);
    atomic_fetch_add(&A->pe, pe);
    atomic_max32(&A->mo, mo);
    atomic_max32(&A->mc, mc);
    free(fs);
    free(view);
}

int port_render_tiles(const port_tree* t, const bt_camera* cam, const bt_render_config* cfg, const uint32_t* offsets,
                      const bt_fragment* frags, int threads, uint8_t* hit, float* depth, uint32_t* evalCount,
                      uint32_t* tmo, uint32_t* tcb, uint8_t* terr, uint64_t* stats6) {
    size_t px = (size_t)cam->width * cam->height;
    uint32_t T = (uint32_t)(((cam->width + 7) / 8) * ((cam->height + 7) / 8));
    memset(hit, 0, px);
    memset(depth, 0, px * 4);
    memset(evalCount, 0, px * 4);
    memset(tmo, 0, T * 4);
    memset(tcb, 0, T * 4);
    memset(terr, 0, T);
    rt_args A = {t, cam, cfg, offsets, frags, hit, depth, evalCount, tmo, tcb, terr, 0, 0, 0, 0, 0};
    parallel_for(T, threads, render_tile, &A);
    if (stats6) {
        stats6[0] = atomic_load(&A.fe);
        stats6[1] = atomic_load(&A.rnv);
        stats6[2] = atomic_load(&A.pe);
        stats6[3] = t->nnodes;
        stats6[4] = atomic_load(&A.mo);
        stats6[5] = atomic_load(&A.mc);
    }
    return 0;
}

/* ---------------------------------------------------------------- normals (tracer.cpp:285-350) */
static v3 grad_normal(const port_tree* t, v3 p, float h) {
    float dx = port_eval_full(t, p.x + h, p.y, p.z) - port_eval_full(t, p.x - h, p.y, p.z);
    float dy = port_eval_full(t, p.x, p.y + h, p.z) - port_eval_full(t, p.x, p.y - h, p.z);
    float dz = port_eval_full(t, p.x, p.y, p.z + h) - port_eval_full(t, p.x, p.y, p.z - h);
    return nrm(V(dx, dy, dz));
}

void port_normals(const port_tree* t, const bt_camera* cam, int mode, const uint8_t* hit, const float* depth,
                  float* normal) {
    int W = cam->width, H = cam->height;
#define HIT(x, y) ((x) >= 0 && (x) < W && (y) >= 0 && (y) < H && hit[(size_t)(y) * W + (x)])
#define POS(x, y) add(pixel_ray(cam, (x), (y)).o, mul(pixel_ray(cam, (x), (y)).d, depth[(size_t)(y) * W + (x)]))
    for (int y = 0; y < H; ++y)
        for (int x = 0; x < W; ++x) {
            size_t i = (size_t)y * W + x;
            v3 n = V(0, 0, 0);
            if (hit[i]) {
                v3 p = POS(x, y);
                float h = fmx(1e-3f, 1e-4f * depth[i]);
                if (mode == 1) {
                    n = grad_normal(t, p, h);
                } else {
                    int l = HIT(x - 1, y), r = HIT(x + 1, y), u = HIT(x, y - 1), d = HIT(x, y + 1);
                    int okX = 1, okY = 1;
                    v3 ddx = V(0, 0, 0), ddy = V(0, 0, 0);
                    if (l && r) ddx = sub(POS(x + 1, y), POS(x - 1, y));
                    else if (r) ddx = sub(POS(x + 1, y), p);
                    else if (l) ddx = sub(p, POS(x - 1, y));
                    else okX = 0;
                    if (u && d) ddy = sub(POS(x, y + 1), POS(x, y - 1));
                    else if (d) ddy = sub(POS(x, y + 1), p);
                    else if (u) ddy = sub(p, POS(x, y - 1));
                    else okY = 0;
                    if (okX && okY) {
                        n = cross(ddx, ddy);
                        float L = len(n);
                        if (L > 1e-12f) {
                            n = dvs(n, L);
                            if (dot(n, pixel_ray(cam, x, y).d) > 0.0f) n = V(-n.x, -n.y, -n.z);
                        } else {
                            okX = 0;
                        }
                    }
                    if (!(okX && okY)) n = grad_normal(t, p, h);
                }
            }
            normal[3 * i] = n.x;
            normal[3 * i + 1] = n.y;
            normal[3 * i + 2] = n.z;
        }
#undef HIT
#undef POS
}

/* ---------------------------------------------------------------- oracle_render (tracer.cpp:238-280) */
typedef struct { const port_tree* t; v3 o, d; } full_ctx;
static float full_field(void* c, float t) {
    full_ctx* k = (full_ctx*)c;
    v3 p = add(k->o, mul(k->d, t));
    return port_eval_full(k->t, p.x, p.y, p.z);
}

typedef struct {
    const port_tree* t;
    const bt_camera* cam;
    const bt_render_config* cfg;
    uint8_t* hit;
    float* depth;
    uint32_t* evalCount;
    _Atomic uint64_t fe;
} or_args;

static void oracle_row(void* p, uint32_t y) {
    or_args* A = (or_args*)p;
    uint64_t fe = 0;
    for (int x = 0; x < A->cam->width; ++x) {
        ray_t R = pixel_ray(A->cam, x, (int)y);
        uint32_t ev = 0;
        float tHit = 0.0f;
        int err = 0;
        full_ctx k = {A->t, R.o, R.d};
        int h = trace(full_field, &k, A->cam->nearZ / R.ddf, A->cam->farZ / R.ddf, A->cfg, &ev, &tHit, &err);
        size_t i = (size_t)y * A->cam->width + x;
        A->evalCount[i] = ev;
        fe += ev;
        A->hit[i] = (uint8_t)h;
        A->depth[i] = h ? tHit : 0.0f;
    }
    atomic_fetch_add(&A->fe, fe);
}

void port_oracle(const port_tree* t, const bt_camera* cam, const bt_render_config* cfg, int threads, uint8_t* hit,
                 float* depth, uint32_t* evalCount, uint64_t* stats6) {
    or_args A = {t, cam, cfg, hit, depth, evalCount, 0};
    parallel_for((uint32_t)cam->height, threads, oracle_row, &A);
    if (stats6) {
        uint64_t fe = atomic_load(&A.fe);
        stats6[0] = fe;
        stats6[1] = fe * t->nnodes;
        stats6[2] = fe * t->nprims;
        stats6[3] = t->nnodes;
        stats6[4] = 0;
        stats6[5] = 0;
    }
}
