/* lfd_oracle.c — plain-C restatement of the reference hot path.  TEST INFRASTRUCTURE ONLY
 * (see lfd_oracle.h).  Every function follows the cited reference lines operation by operation,
 * in the reference's evaluation order, with no shortcuts (the GPU's exact-identity shortcuts are
 * therefore checked independently).  Build: -O3 -ffp-contract=off (oracle/Makefile); exp / expf /
 * sqrt / lround / floor come from the host glibc, like the reference's.
 */
#include "lfd_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ primitives -------- */

typedef struct {
    double K[9], R[9], t[3];
} cam_t; /* PinholeCamera (geometry.hpp:22), row-major */

static cam_t cam_at(const double* cams, int v) {
    cam_t c;
    memcpy(c.K, cams + 21 * v, 9 * sizeof(double));
    memcpy(c.R, cams + 21 * v + 9, 9 * sizeof(double));
    memcpy(c.t, cams + 21 * v + 18, 3 * sizeof(double));
    return c;
}

/* PinholeCamera::ray (geometry.hpp:45-50) */
static void ray(const cam_t* c, double px, double py, double r[3]) {
    const double y = (py - c->K[5]) / c->K[4];
    const double x = (px - c->K[2] - c->K[1] * y) / c->K[0];
    r[0] = x;
    r[1] = y;
    r[2] = 1.0;
}

static double dot3(const double a[3], const double b[3]) { return a[0] * b[0] + a[1] * b[1] + a[2] * b[2]; }

/* color_dist2 (image.hpp:13-16) */
static float color_dist2(const float* a, const float* b) {
    const float d0 = a[0] - b[0], d1 = a[1] - b[1], d2 = a[2] - b[2];
    return d0 * d0 + d1 * d1 + d2 * d2;
}

/* plane_depth_at (geometry.hpp:85-92): returns 0 and leaves *out when degenerate */
static int plane_depth_at(const cam_t* c, const double pl[4], double cx, double cy, double qx, double qy,
                          double* out) {
    double rc[3], v[3];
    ray(c, cx, cy, rc);
    const double anchor[3] = {pl[0] * rc[0], pl[0] * rc[1], pl[0] * rc[2]};
    ray(c, qx, qy, v);
    const double n[3] = {pl[1], pl[2], pl[3]};
    const double denom = dot3(n, v);
    if (fabs(denom) <= 1e-9) return 0;
    *out = dot3(n, anchor) / denom;
    return 1;
}

/* ImageBuffer::contains / bilinear (image.hpp:42-67) */
static int contains(int W, int H, double x, double y) { return x >= 0.0 && y >= 0.0 && x <= W - 1.0 && y <= H - 1.0; }

static void bilinear(const float* img, int W, int H, double x, double y, float out[3]) {
    int x0 = (int)floor(x);
    int y0 = (int)floor(y);
    if (x0 >= W - 1) x0 = W - 2;
    if (y0 >= H - 1) y0 = H - 2;
    if (x0 < 0) x0 = 0;
    if (y0 < 0) y0 = 0;
    const float fx = (float)(x - x0);
    const float fy = (float)(y - y0);
    const float* p00 = img + ((size_t)y0 * W + x0) * 3;
    const float* p10 = p00 + 3;
    const float* p01 = p00 + (size_t)W * 3;
    const float* p11 = p01 + 3;
    for (int c = 0; c < 3; ++c) {
        const float top = p00[c] + fx * (p10[c] - p00[c]);
        const float bot = p01[c] + fx * (p11[c] - p01[c]);
        out[c] = top + fy * (bot - top);
    }
}

/* RandomStream / derive_stream (rng.hpp:9-39) */
static uint64_t next_u64(uint64_t* s) {
    uint64_t z = (*s += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
static double next_double(uint64_t* s) { return (double)(next_u64(s) >> 11) * 0x1.0p-53; }
static uint64_t derive_stream(uint64_t seed, uint64_t view, uint64_t sp) {
    uint64_t h = seed;
    h ^= (view + 0x9E3779B97F4A7C15ull + (h << 6) + (h >> 2));
    h *= 0xFF51AFD7ED558CCDull;
    h ^= (sp + 0x9E3779B97F4A7C15ull + (h << 6) + (h >> 2));
    h *= 0xC4CEB9FE1A85EC53ull;
    h ^= h >> 33;
    return h;
}

/* ------------------------------------------------------------------ SLIC ------------- */

/* recompute_stats (superpixel.hpp:55-83) */
static void recompute_stats(const float* img, lfdo_grid* g) {
    const int n = g->gw * g->gh;
    double* sx = calloc((size_t)n * 5, sizeof(double));
    double *sy = sx + n, *s0 = sy + n, *s1 = s0 + n, *s2 = s1 + n;
    int* cnt = calloc(n, sizeof(int));
    for (int y = 0; y < g->H; ++y)
        for (int x = 0; x < g->W; ++x) {
            const int id = g->labels[y * g->W + x];
            const float* c = img + ((size_t)y * g->W + x) * 3;
            sx[id] += x;
            sy[id] += y;
            s0[id] += c[0];
            s1[id] += c[1];
            s2[id] += c[2];
            ++cnt[id];
        }
    /* member lists (grid.pixels) as CSR, row-major per superpixel */
    g->off[0] = 0;
    for (int id = 0; id < n; ++id) g->off[id + 1] = g->off[id] + cnt[id];
    int* cur = malloc(n * sizeof(int));
    memcpy(cur, g->off, n * sizeof(int));
    for (int p = 0; p < g->W * g->H; ++p) g->mem[cur[g->labels[p]]++] = p;
    for (int id = 0; id < n; ++id) {
        lfdo_record* r = &g->rec[id];
        r->count = cnt[id];
        r->gx = id % g->gw;
        r->gy = id / g->gw;
        if (cnt[id] > 0) {
            r->cx = sx[id] / cnt[id];
            r->cy = sy[id] / cnt[id];
            r->color[0] = (float)(s0[id] / cnt[id]);
            r->color[1] = (float)(s1[id] / cnt[id]);
            r->color[2] = (float)(s2[id] / cnt[id]);
        } else {
            r->cx = r->cy = 0;
            r->color[0] = r->color[1] = r->color[2] = 0.f;
        }
    }
    free(cur);
    free(cnt);
    free(sx);
}

/* detail::enforce_connectivity (superpixel.hpp:87-172) */
static void enforce_connectivity(lfdo_grid* g) {
    const int w = g->W, h = g->H, npx = w * h, n = g->gw * g->gh;
    int* comp = malloc(npx * sizeof(int));
    for (int i = 0; i < npx; ++i) comp[i] = -1;
    int* clabel = malloc(npx * sizeof(int));   /* per component */
    int* cstart = malloc((npx + 1) * sizeof(int));
    int* cpix = malloc(npx * sizeof(int));     /* component pixels, in DFS pop order */
    int* stack = malloc(npx * sizeof(int));
    const int dx4[4] = {1, -1, 0, 0}, dy4[4] = {0, 0, 1, -1};
    int ncomp = 0, fill = 0;
    for (int i = 0; i < npx; ++i) {
        if (comp[i] >= 0) continue;
        const int cid = ncomp++;
        clabel[cid] = g->labels[i];
        cstart[cid] = fill;
        int sp = 0;
        stack[sp++] = i;
        comp[i] = cid;
        while (sp > 0) {
            const int p = stack[--sp];
            cpix[fill++] = p;
            const int px = p % w, py = p / w;
            for (int k = 0; k < 4; ++k) {
                const int nx = px + dx4[k], ny = py + dy4[k];
                if (nx < 0 || ny < 0 || nx >= w || ny >= h) continue;
                const int q = ny * w + nx;
                if (comp[q] < 0 && g->labels[q] == clabel[cid]) {
                    comp[q] = cid;
                    stack[sp++] = q;
                }
            }
        }
    }
    cstart[ncomp] = fill;
    int* keeper = malloc(n * sizeof(int));
    for (int l = 0; l < n; ++l) keeper[l] = -1;
    for (int c = 0; c < ncomp; ++c) {
        const int lab = clabel[c];
        const int sz = cstart[c + 1] - cstart[c];
        if (keeper[lab] < 0 || sz > cstart[keeper[lab] + 1] - cstart[keeper[lab]]) keeper[lab] = c;
    }
    int* count = calloc(n, sizeof(int));
    char* assigned = calloc(ncomp, 1);
    int* merged = malloc(ncomp * sizeof(int));
    for (int c = 0; c < ncomp; ++c) {
        merged[c] = clabel[c];
        if (c == keeper[clabel[c]]) {
            assigned[c] = 1;
            count[clabel[c]] += cstart[c + 1] - cstart[c];
        }
    }
    int progress = 1;
    while (progress) {
        progress = 0;
        int pending = 0;
        for (int c = 0; c < ncomp; ++c) {
            if (assigned[c]) continue;
            int best = -1;
            for (int k0 = cstart[c]; k0 < cstart[c + 1]; ++k0) {
                const int p = cpix[k0];
                const int px = p % w, py = p / w;
                for (int k = 0; k < 4; ++k) {
                    const int nx = px + dx4[k], ny = py + dy4[k];
                    if (nx < 0 || ny < 0 || nx >= w || ny >= h) continue;
                    const int nc = comp[ny * w + nx];
                    if (nc == c || !assigned[nc]) continue;
                    const int nl = merged[nc];
                    if (best < 0 || count[nl] > count[best] || (count[nl] == count[best] && nl < best)) best = nl;
                }
            }
            if (best < 0) {
                pending = 1;
                continue;
            }
            merged[c] = best;
            assigned[c] = 1;
            progress = 1;
            for (int k0 = cstart[c]; k0 < cstart[c + 1]; ++k0) g->labels[cpix[k0]] = best;
            count[best] += cstart[c + 1] - cstart[c];
        }
        if (!pending) break;
    }
    free(comp);
    free(clabel);
    free(cstart);
    free(cpix);
    free(stack);
    free(keeper);
    free(count);
    free(assigned);
    free(merged);
}

int lfdo_slic_segment(int W, int H, const float* img, int S, float compactness, int iterations, lfdo_grid* g) {
    if (S < 4 || !(compactness > 0) || iterations < 1) return 1; /* SlicParams::validate */
    if (W < S || H < S) return 1;
    g->W = W;
    g->H = H;
    g->S = S;
    g->gw = (W + S - 1) / S;
    g->gh = (H + S - 1) / S;
    const int n = g->gw * g->gh;
    double* ccx = malloc(n * sizeof(double));
    double* ccy = malloc(n * sizeof(double));
    float* ccol = malloc((size_t)n * 3 * sizeof(float));
    /* centre init (superpixel.hpp:202-213) */
    for (int gy = 0; gy < g->gh; ++gy)
        for (int gx = 0; gx < g->gw; ++gx) {
            const int x0 = gx * S, x1 = W < x0 + S ? W : x0 + S;
            const int y0 = gy * S, y1 = H < y0 + S ? H : y0 + S;
            const int id = gy * g->gw + gx;
            ccx[id] = 0.5 * (x0 + x1 - 1);
            ccy[id] = 0.5 * (y0 + y1 - 1);
            memcpy(ccol + 3 * id, img + ((size_t)(int)ccy[id] * W + (int)ccx[id]) * 3, 3 * sizeof(float));
        }
    const float spatial_w = compactness / (float)S;
    double* sums = malloc((size_t)n * 5 * sizeof(double));
    int* cnt = malloc(n * sizeof(int));
    for (int it = 0; it < iterations; ++it) {
        /* assignment (superpixel.hpp:219-245) */
        for (int y = 0; y < H; ++y)
            for (int x = 0; x < W; ++x) {
                const float* pc = img + ((size_t)y * W + x) * 3;
                const int pgx = x / S, pgy = y / S;
                float best_d = 0, best_s = 0;
                int best = -1;
                const int gy0 = pgy - 2 > 0 ? pgy - 2 : 0, gy1 = pgy + 2 < g->gh - 1 ? pgy + 2 : g->gh - 1;
                const int gx0 = pgx - 2 > 0 ? pgx - 2 : 0, gx1 = pgx + 2 < g->gw - 1 ? pgx + 2 : g->gw - 1;
                for (int gy = gy0; gy <= gy1; ++gy)
                    for (int gx = gx0; gx <= gx1; ++gx) {
                        const int id = gy * g->gw + gx;
                        const double ddx = x - ccx[id], ddy = y - ccy[id];
                        const float ds = (float)sqrt(ddx * ddx + ddy * ddy);
                        if (ds > 2.f * S) continue;
                        const float dc = sqrtf(color_dist2(pc, ccol + 3 * id));
                        const float d = dc + spatial_w * ds;
                        if (best < 0 || d < best_d || (d == best_d && ds < best_s)) {
                            best_d = d;
                            best_s = ds;
                            best = id;
                        }
                    }
                g->labels[y * W + x] = best;
            }
        /* update (superpixel.hpp:246-267) */
        memset(sums, 0, (size_t)n * 5 * sizeof(double));
        memset(cnt, 0, n * sizeof(int));
        for (int y = 0; y < H; ++y)
            for (int x = 0; x < W; ++x) {
                const int id = g->labels[y * W + x];
                const float* c = img + ((size_t)y * W + x) * 3;
                sums[5 * id] += x;
                sums[5 * id + 1] += y;
                sums[5 * id + 2] += c[0];
                sums[5 * id + 3] += c[1];
                sums[5 * id + 4] += c[2];
                ++cnt[id];
            }
        for (int id = 0; id < n; ++id) {
            if (cnt[id] == 0) continue;
            ccx[id] = sums[5 * id] / cnt[id];
            ccy[id] = sums[5 * id + 1] / cnt[id];
            ccol[3 * id] = (float)(sums[5 * id + 2] / cnt[id]);
            ccol[3 * id + 1] = (float)(sums[5 * id + 3] / cnt[id]);
            ccol[3 * id + 2] = (float)(sums[5 * id + 4] / cnt[id]);
        }
    }
    enforce_connectivity(g);
    /* empty-cluster repair (superpixel.hpp:272-308) */
    memset(cnt, 0, n * sizeof(int));
    for (int p = 0; p < W * H; ++p) ++cnt[g->labels[p]];
    char* seen = malloc((size_t)W * H);
    int* queue = malloc((size_t)W * H * sizeof(int));
    for (int id = 0; id < n; ++id) {
        if (cnt[id] > 0) continue;
        const int gx = id % g->gw, gy = id / g->gw;
        const int x = W - 1 < gx * S + S / 2 ? W - 1 : gx * S + S / 2;
        const int y = H - 1 < gy * S + S / 2 ? H - 1 : gy * S + S / 2;
        const int old = g->labels[y * W + x];
        if (cnt[old] > 1) {
            memset(seen, 0, (size_t)W * H);
            int head = 0, tail = 0;
            queue[tail++] = y * W + x;
            seen[queue[0]] = 1;
            int last = queue[0];
            for (; head < tail; ++head) {
                last = queue[head];
                const int px = last % W, py = last / W;
                const int nb[4][2] = {{px + 1, py}, {px - 1, py}, {px, py + 1}, {px, py - 1}};
                for (int k = 0; k < 4; ++k) {
                    if (nb[k][0] < 0 || nb[k][1] < 0 || nb[k][0] >= W || nb[k][1] >= H) continue;
                    const int qi = nb[k][1] * W + nb[k][0];
                    if (!seen[qi] && g->labels[qi] == old) {
                        seen[qi] = 1;
                        queue[tail++] = qi;
                    }
                }
            }
            g->labels[last] = id;
            --cnt[old];
            cnt[id] = 1;
        }
    }
    free(seen);
    free(queue);
    recompute_stats(img, g);
    free(ccx);
    free(ccy);
    free(ccol);
    free(sums);
    free(cnt);
    return 0;
}

/* ------------------------------------------------------------------ sweep ------------ */

static void center(const cam_t* c, double out[3]) { /* -R^T t (geometry.hpp:41) */
    for (int i = 0; i < 3; ++i) out[i] = (-c->R[0 * 3 + i]) * c->t[0] + (-c->R[1 * 3 + i]) * c->t[1] + (-c->R[2 * 3 + i]) * c->t[2];
}

/* matching_views (sweep.hpp:67-80); returns the count */
static int matching_views(int V, const double* cams, int view, int max_nb, int* out) {
    int n = 0;
    for (int i = 0; i < V; ++i)
        if (i != view) out[n++] = i;
    if (max_nb > 0 && n > max_nb) {
        double cv[3], d[64 * 64];
        const cam_t c0 = cam_at(cams, view);
        center(&c0, cv);
        for (int k = 0; k < n; ++k) {
            double ck[3];
            const cam_t ci = cam_at(cams, out[k]);
            center(&ci, ck);
            const double a = ck[0] - cv[0], b = ck[1] - cv[1], e = ck[2] - cv[2];
            d[out[k]] = a * a + b * b + e * e;
        }
        for (int i = 1; i < n; ++i) { /* stable insertion sort by distance */
            const int key = out[i];
            int j = i - 1;
            while (j >= 0 && d[key] < d[out[j]]) {
                out[j + 1] = out[j];
                --j;
            }
            out[j + 1] = key;
        }
        n = max_nb;
        for (int i = 1; i < n; ++i) { /* sort ids ascending */
            const int key = out[i];
            int j = i - 1;
            while (j >= 0 && out[j] > key) {
                out[j + 1] = out[j];
                --j;
            }
            out[j + 1] = key;
        }
    }
    return n;
}

/* map_pixel_via_plane (geometry.hpp:102-111) */
static int map_pixel(const cam_t* ref, const double pl[4], double cx, double cy, double x, double y, const cam_t* tg,
                     double* u, double* v) {
    double d;
    if (!plane_depth_at(ref, pl, cx, cy, x, y, &d)) return 0;
    double r[3];
    ray(ref, x, y, r);
    const double a[3] = {d * r[0] - ref->t[0], d * r[1] - ref->t[1], d * r[2] - ref->t[2]};
    double wv[3], cp[3], hv[3];
    for (int i = 0; i < 3; ++i) wv[i] = ref->R[0 * 3 + i] * a[0] + ref->R[1 * 3 + i] * a[1] + ref->R[2 * 3 + i] * a[2];
    for (int i = 0; i < 3; ++i) cp[i] = tg->R[i * 3] * wv[0] + tg->R[i * 3 + 1] * wv[1] + tg->R[i * 3 + 2] * wv[2] + tg->t[i];
    for (int i = 0; i < 3; ++i) hv[i] = tg->K[i * 3] * cp[0] + tg->K[i * 3 + 1] * cp[1] + tg->K[i * 3 + 2] * cp[2];
    *u = hv[0] / hv[2];
    *v = hv[1] / hv[2];
    return !(cp[2] <= 0);
}

/* sweep_cost (sweep.hpp:85-107) */
static double sweep_cost(int W, int H, const float* images, const double* cams, const lfdo_grid* g, int view, int sp,
                         double depth, const int* targets, int nt, float T) {
    const cam_t rc = cam_at(cams, view);
    const double pl[4] = {depth, 0, 0, -1};
    const double cx = g->rec[sp].cx, cy = g->rec[sp].cy;
    const float* rimg = images + (size_t)view * W * H * 3;
    double cost = 0;
    for (int k = 0; k < nt; ++k) {
        const cam_t tc = cam_at(cams, targets[k]);
        const float* timg = images + (size_t)targets[k] * W * H * 3;
        for (int m = g->off[sp]; m < g->off[sp + 1]; ++m) {
            const int p = g->mem[m];
            const int x = p % W, y = p / W;
            double u, v;
            if (!map_pixel(&rc, pl, cx, cy, x, y, &tc, &u, &v) || !contains(W, H, u, v)) {
                cost += T;
                continue;
            }
            float out[3];
            bilinear(timg, W, H, u, v, out);
            const float d2 = color_dist2(rimg + (size_t)p * 3, out);
            cost += d2 < T ? d2 : T; /* tssd: std::min(T, dist2) */
        }
    }
    return cost;
}

int lfdo_sweep_view(int V, const float* images, const double* cams, double d_min, double d_max, const lfdo_grid* grids,
                    int view, int levels, float threshold, int max_neighbors, uint64_t seed, double* planes_out) {
    if (levels < 2 || !(threshold > 0)) return 1;
    if (!(0 < d_min && d_min < d_max)) return 2;
    const lfdo_grid* g = &grids[view];
    int targets[64];
    const int nt = matching_views(V, cams, view, max_neighbors, targets);
    double* depths = malloc(levels * sizeof(double));
    for (int sp = 0; sp < g->gw * g->gh; ++sp) {
        uint64_t st = derive_stream(seed, (uint64_t)view, (uint64_t)sp);
        const double inv_lo = 1.0 / d_max, inv_hi = 1.0 / d_min; /* sample_inverse_depths (geometry.hpp:116-130) */
        const double step = (inv_hi - inv_lo) / (levels - 1);
        for (int k = 0; k < levels; ++k) {
            double inv = inv_lo + step * k + next_double(&st) * step;
            if (inv > inv_hi) inv = inv_hi;
            depths[k] = 1.0 / inv;
        }
        double best_c = 0, best_d = 0;
        int first = 1;
        for (int k = levels - 1; k >= 0; --k) {
            const double c = sweep_cost(g->W, g->H, images, cams, g, view, sp, depths[k], targets, nt, threshold);
            if (first || c < best_c || (c == best_c && depths[k] < best_d)) {
                best_c = c;
                best_d = depths[k];
                first = 0;
            }
        }
        planes_out[4 * sp] = best_d;
        planes_out[4 * sp + 1] = 0.0;
        planes_out[4 * sp + 2] = 0.0;
        planes_out[4 * sp + 3] = -1.0;
    }
    free(depths);
    return 0;
}

/* rasterize (sweep.hpp:44-63) for one view */
void lfdo_rasterize(const double* cam, const lfdo_grid* g, const double* planes, float* depth_out) {
    cam_t c;
    memcpy(c.K, cam, 9 * sizeof(double));
    memcpy(c.R, cam + 9, 9 * sizeof(double));
    memcpy(c.t, cam + 18, 3 * sizeof(double));
    for (int p = 0; p < g->W * g->H; ++p) depth_out[p] = 0.f;
    for (int sp = 0; sp < g->gw * g->gh; ++sp) {
        const double* pl = planes + 4 * sp;
        double rc[3];
        ray(&c, g->rec[sp].cx, g->rec[sp].cy, rc);
        const double anchor[3] = {pl[0] * rc[0], pl[0] * rc[1], pl[0] * rc[2]};
        const double n[3] = {pl[1], pl[2], pl[3]};
        const double num = dot3(n, anchor);
        for (int m = g->off[sp]; m < g->off[sp + 1]; ++m) {
            const int p = g->mem[m];
            double v[3];
            ray(&c, p % g->W, p / g->W, v);
            const double denom = dot3(n, v);
            depth_out[p] = fabs(denom) <= 1e-9 ? 0.f : (float)(num / denom);
        }
    }
}

/* ------------------------------------------------------------------ refinement ------- */

static const int kDir[8][2] = {{1, 0}, {1, -1}, {0, -1}, {-1, -1}, {-1, 0}, {-1, 1}, {0, 1}, {1, 1}};

typedef struct {
    int V;
    const double* cams;
    double d_min, d_max;
    const lfdo_grid* grids;
    const lfdo_energy* p;
    const double* planes; /* snapshot [V][nsp][4] */
    const float* depth;   /* snapshot [V][H*W] */
    int targets[64][64];
    int nt[64];
    double rel[64][64][12]; /* rel_rot (row-major) + rel_trans, indexed [v][t] */
    float* min_nb_sim;      /* [V][nsp] */
} ctx_t;

/* color_similarity (superpixel.hpp:346-348) */
static float color_similarity(const float* a, const float* b, float alpha) {
    return expf(-color_dist2(a, b) / (2.f * alpha * alpha));
}

/* depth_consistency (refine.hpp:34-37) */
static double depth_consistency(double d1, double d2, double sigma) {
    const double r = 1.0 / d1 - 1.0 / d2;
    return exp(-(r * r) / (2.0 * sigma * sigma));
}

/* smoothness_term (refine.hpp:84-100) */
static double smoothness_term(const ctx_t* c, int v, int sp, const double pl[4]) {
    const lfdo_grid* g = &c->grids[v];
    const cam_t cam = cam_at(c->cams, v);
    const int nsp = g->gw * g->gh;
    const int gx = sp % g->gw, gy = sp / g->gw;
    double wsum = 0, acc = 0;
    for (int k = 0; k < 8; ++k) {
        const int nx = gx + kDir[k][0], ny = gy + kDir[k][1];
        if (nx < 0 || ny < 0 || nx >= g->gw || ny >= g->gh) continue;
        const int nb = ny * g->gw + nx;
        const double w = color_similarity(g->rec[sp].color, g->rec[nb].color, c->p->alpha);
        wsum += w;
        double ext;
        if (!plane_depth_at(&cam, pl, g->rec[sp].cx, g->rec[sp].cy, g->rec[nb].cx, g->rec[nb].cy, &ext) || ext <= 0)
            continue;
        acc += w * depth_consistency(c->planes[((size_t)v * nsp + nb) * 4], ext, c->p->sigma);
    }
    if (wsum <= 1e-30) return 1.0;
    return acc / wsum;
}

/* pair_stats (refine.hpp:111-172) -> visibility + occlusion */
static double pair_vo(const ctx_t* c, int v, int sp, const double pl[4], int t) {
    const lfdo_grid* g = &c->grids[v];
    const lfdo_grid* tg = &c->grids[t];
    const cam_t cam = cam_at(c->cams, v);
    const cam_t tcam = cam_at(c->cams, t);
    const double* R = c->rel[v][t];
    const double* tr = R + 9;
    const float* tdepth = c->depth + (size_t)t * tg->W * tg->H;
    const float* ref_color = g->rec[sp].color;
    double rc[3];
    ray(&cam, g->rec[sp].cx, g->rec[sp].cy, rc);
    const double anchor[3] = {pl[0] * rc[0], pl[0] * rc[1], pl[0] * rc[2]};
    const double n[3] = {pl[1], pl[2], pl[3]};
    const double plane_num = dot3(n, anchor);
    const double inv_two_sigma2 = 1.0 / (2.0 * c->p->sigma * c->p->sigma);
    const double inv_two_alpha2 = 1.0 / (2.0 * (double)c->p->alpha * c->p->alpha);
    double photo_sum = 0, vis_sum = 0;
    int x_count = 0, y_nonempty = 0, cached_label = -1;
    double cached_w = 0;
    for (int m = g->off[sp]; m < g->off[sp + 1]; ++m) {
        const int p = g->mem[m];
        double vr[3];
        ray(&cam, p % g->W, p / g->W, vr);
        const double denom = dot3(n, vr);
        if (fabs(denom) <= 1e-9) continue;
        const double s = plane_num / denom;
        if (s <= 0) continue;
        const double sv[3] = {s * vr[0], s * vr[1], s * vr[2]};
        double xt[3];
        for (int i = 0; i < 3; ++i) xt[i] = R[i * 3] * sv[0] + R[i * 3 + 1] * sv[1] + R[i * 3 + 2] * sv[2] + tr[i];
        if (xt[2] <= 0) continue;
        const double u = (tcam.K[0] * xt[0] + tcam.K[1] * xt[1] + tcam.K[2] * xt[2]) / xt[2];
        const double w = (tcam.K[4] * xt[1] + tcam.K[5] * xt[2]) / xt[2];
        const int px = (int)lround(u);
        const int py = (int)lround(w);
        if (px < 0 || py < 0 || px >= tg->W || py >= tg->H) continue;
        const int tlab = tg->labels[py * tg->W + px];
        if (tlab != cached_label) {
            cached_label = tlab;
            cached_w = exp(-(double)color_dist2(ref_color, tg->rec[tlab].color) * inv_two_alpha2);
        }
        photo_sum += cached_w;
        const float td = tdepth[py * tg->W + px];
        if (td <= 0) continue;
        if (xt[2] <= td * (1.0 + 1e-6)) {
            const double r = 1.0 / xt[2] - 1.0 / td;
            vis_sum += exp(-r * r * inv_two_sigma2);
            ++x_count;
        } else {
            y_nonempty = 1;
        }
    }
    const double photo = photo_sum / (double)(g->off[sp + 1] - g->off[sp]);
    const double vis = x_count > 0 ? photo * (vis_sum / x_count) : 0.0;
    double occ = 0.0;
    if (c->p->use_occlusion && y_nonempty) occ = c->p->eta * (1.0 - c->min_nb_sim[(size_t)v * (g->gw * g->gh) + sp]);
    return vis + occ;
}

/* consistency_term (refine.hpp:189-199) */
static double consistency_term(const ctx_t* c, int v, int sp, const double pl[4]) {
    if (c->nt[v] == 0) return 1.0;
    double acc = 0;
    for (int k = 0; k < c->nt[v]; ++k) acc += pair_vo(c, v, sp, pl, c->targets[v][k]);
    return acc / (double)c->nt[v];
}

/* energy (refine.hpp:201-207) */
static double energy(const ctx_t* c, int v, int sp, const double pl[4]) {
    double e = 1.0;
    if (c->p->use_smoothness) e *= smoothness_term(c, v, sp, pl);
    if (c->p->use_consistency) e *= consistency_term(c, v, sp, pl);
    return e;
}

/* normal_candidates (refine.hpp:213-242); returns the count */
static int normal_candidates(const ctx_t* c, int v, int sp, double out[8][3]) {
    const lfdo_grid* g = &c->grids[v];
    const cam_t cam = cam_at(c->cams, v);
    const int nsp = g->gw * g->gh;
    const int gx = sp % g->gw, gy = sp / g->gw;
    int ring[8];
    for (int k = 0; k < 8; ++k) {
        const int nx = gx + kDir[k][0], ny = gy + kDir[k][1];
        ring[k] = (nx < 0 || ny < 0 || nx >= g->gw || ny >= g->gh) ? -1 : ny * g->gw + nx;
    }
#define LIFT(id, o)                                                          \
    do {                                                                     \
        double r_[3];                                                        \
        ray(&cam, g->rec[id].cx, g->rec[id].cy, r_);                         \
        const double d_ = c->planes[((size_t)v * nsp + (id)) * 4];           \
        (o)[0] = d_ * r_[0];                                                 \
        (o)[1] = d_ * r_[1];                                                 \
        (o)[2] = d_ * r_[2];                                                 \
    } while (0)
    double ref_pt[3], ref_ray[3];
    LIFT(sp, ref_pt);
    ray(&cam, g->rec[sp].cx, g->rec[sp].cy, ref_ray);
    int cnt = 0;
    for (int k = 0; k < 8; ++k) {
        const int a = ring[k], b = ring[(k + 1) % 8];
        if (a < 0 || b < 0) continue;
        double la[3], lb[3];
        LIFT(a, la);
        LIFT(b, lb);
        const double A[3] = {la[0] - ref_pt[0], la[1] - ref_pt[1], la[2] - ref_pt[2]};
        const double B[3] = {lb[0] - ref_pt[0], lb[1] - ref_pt[1], lb[2] - ref_pt[2]};
        double nrm[3] = {A[1] * B[2] - A[2] * B[1], A[2] * B[0] - A[0] * B[2], A[0] * B[1] - A[1] * B[0]};
        const double len = sqrt(nrm[0] * nrm[0] + nrm[1] * nrm[1] + nrm[2] * nrm[2]);
        if (len <= 1e-12) continue;
        for (int i = 0; i < 3; ++i) nrm[i] = nrm[i] / len;
        if (dot3(nrm, ref_ray) > 0)
            for (int i = 0; i < 3; ++i) nrm[i] = -nrm[i];
        if (dot3(nrm, ref_ray) >= 0) continue;
        memcpy(out[cnt++], nrm, sizeof(nrm));
    }
#undef LIFT
    return cnt;
}

int lfdo_refine_iteration(int V, const double* cams, double d_min, double d_max, const lfdo_grid* grids,
                          const lfdo_energy* p, const double* planes_all, const float* depth_all, int l,
                          double* planes_out, uint64_t* accepted) {
    if (V > 64) return 1;
    ctx_t* c = calloc(1, sizeof(ctx_t));
    c->V = V;
    c->cams = cams;
    c->d_min = d_min;
    c->d_max = d_max;
    c->grids = grids;
    c->p = p;
    c->planes = planes_all;
    c->depth = depth_all;
    /* make_refine_context tables (refine.hpp:67-77) */
    size_t total = 0;
    for (int v = 0; v < V; ++v) total += (size_t)grids[v].gw * grids[v].gh;
    c->min_nb_sim = malloc(total * sizeof(float));
    for (int v = 0; v < V; ++v) {
        c->nt[v] = matching_views(V, cams, v, p->max_neighbors, c->targets[v]);
        const lfdo_grid* g = &grids[v];
        for (int sp = 0; sp < g->gw * g->gh; ++sp) { /* min_neighbor_similarity (superpixel.hpp:352-357) */
            float m = 1.f;
            const int gx = sp % g->gw, gy = sp / g->gw;
            for (int k = 0; k < 8; ++k) {
                const int nx = gx + kDir[k][0], ny = gy + kDir[k][1];
                if (nx < 0 || ny < 0 || nx >= g->gw || ny >= g->gh) continue;
                const float s = color_similarity(g->rec[sp].color, g->rec[ny * g->gw + nx].color, p->alpha);
                m = s < m ? s : m;
            }
            c->min_nb_sim[(size_t)v * (g->gw * g->gh) + sp] = m;
        }
        const cam_t cv = cam_at(cams, v);
        for (int t = 0; t < V; ++t) {
            if (t == v) continue;
            const cam_t ct = cam_at(cams, t);
            double* r = c->rel[v][t];
            for (int a = 0; a < 3; ++a)
                for (int b = 0; b < 3; ++b)
                    r[a * 3 + b] = ct.R[a * 3] * cv.R[b * 3] + ct.R[a * 3 + 1] * cv.R[b * 3 + 1] + ct.R[a * 3 + 2] * cv.R[b * 3 + 2];
            for (int a = 0; a < 3; ++a)
                r[9 + a] = ct.t[a] - (r[a * 3] * cv.t[0] + r[a * 3 + 1] * cv.t[1] + r[a * 3 + 2] * cv.t[2]);
        }
    }
    /* refine_iteration (refine.hpp:253-323) */
    const int kernel_px = (int)(p->size_init / (double)l);
    const int ks = (int)lround(p->steps_init / (double)l);
    const int kernel_step = ks > 1 ? ks : 1;
    const double max_consistency = p->use_occlusion ? 1.0 + p->eta : 1.0;
    uint64_t acc = 0;
    size_t base = 0;
    for (int v = 0; v < V; ++v) {
        const lfdo_grid* g = &grids[v];
        const int nsp = g->gw * g->gh;
        const cam_t cam = cam_at(cams, v);
        /* grid_neighbors(Kernel) (superpixel.hpp:318-343) */
        const int radius_sp = kernel_px / (g->S > 1 ? g->S : 1);
        int* nbs = malloc((8 + 8 * (radius_sp / kernel_step + 1)) * sizeof(int));
        for (int sp = 0; sp < nsp; ++sp) {
            const int gx = sp % g->gw, gy = sp / g->gw;
            int nn = 0;
            for (int k = 0; k < 8; ++k) {
                const int nx = gx + kDir[k][0], ny = gy + kDir[k][1];
                if (nx < 0 || ny < 0 || nx >= g->gw || ny >= g->gh) continue;
                nbs[nn++] = ny * g->gw + nx;
            }
            for (int k = 0; k < 8; ++k)
                for (int r = kernel_step; r <= radius_sp; r += kernel_step) {
                    if (abs(kDir[k][0]) * r <= 1 && abs(kDir[k][1]) * r <= 1) continue;
                    const int nx = gx + kDir[k][0] * r, ny = gy + kDir[k][1] * r;
                    if (nx < 0 || ny < 0 || nx >= g->gw || ny >= g->gh) continue;
                    const int id = ny * g->gw + nx;
                    int dup = 0;
                    for (int q = 0; q < nn; ++q) dup |= nbs[q] == id;
                    if (!dup) nbs[nn++] = id;
                }
            double cur[4];
            memcpy(cur, planes_all + ((size_t)v * nsp + sp) * 4, sizeof(cur));
            double e_cur = energy(c, v, sp, cur);
#define TRY(cand)                                                                                         \
    do {                                                                                                  \
        if (!((cand)[0] == cur[0] && (cand)[1] == cur[1] && (cand)[2] == cur[2] && (cand)[3] == cur[3]) && \
            !((cand)[0] < d_min || (cand)[0] > d_max)) {                                                  \
            double e_;                                                                                    \
            int eval_ = 1;                                                                                \
            if (p->use_smoothness && p->use_consistency) {                                                \
                const double es_ = smoothness_term(c, v, sp, cand);                                       \
                if (es_ * max_consistency <= e_cur) eval_ = 0;                                            \
                else e_ = es_ * consistency_term(c, v, sp, cand);                                         \
            } else {                                                                                      \
                e_ = energy(c, v, sp, cand);                                                              \
            }                                                                                             \
            if (eval_ && e_ > e_cur) {                                                                    \
                ++acc;                                                                                    \
                memcpy(cur, cand, sizeof(cur));                                                           \
                e_cur = e_;                                                                               \
            }                                                                                             \
        }                                                                                                 \
    } while (0)
            for (int q = 0; q < nn; ++q) { /* propagation (refine.hpp:307-314) */
                const int nb = nbs[q];
                const double* np = planes_all + ((size_t)v * nsp + nb) * 4;
                double d;
                if (!plane_depth_at(&cam, np, g->rec[nb].cx, g->rec[nb].cy, g->rec[sp].cx, g->rec[sp].cy, &d) || d <= 0)
                    continue;
                const double cand[4] = {d, np[1], np[2], np[3]};
                TRY(cand);
            }
            double normals[8][3]; /* normal refinement (refine.hpp:317-318) */
            const int nn2 = normal_candidates(c, v, sp, normals);
            for (int q = 0; q < nn2; ++q) {
                const double cand[4] = {cur[0], normals[q][0], normals[q][1], normals[q][2]};
                TRY(cand);
            }
#undef TRY
            memcpy(planes_out + (base + sp) * 4, cur, sizeof(cur));
        }
        free(nbs);
        base += nsp;
    }
    if (accepted) *accepted = acc;
    free(c->min_nb_sim);
    free(c);
    return 0;
}
