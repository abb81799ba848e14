/*
 * dpm_oracle.c -- CPU restatement of the reference DPM hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker (and the
 * bench.py `cpu_baseline` / `--impl reference` port).  The product path in
 * paper_2012_08099_b200/ never links, loads or calls it.
 *
 * What it restates (reference = /root/reference, read-only):
 *   - projection index maps           pkg/src/volmoments/projection.py:7-14, 139-191
 *                                      pkg/tests/conftest.py:11-37 (oracle_project)
 *   - 2D raw moments about a logical  pkg/src/volmoments/drt2d.py:177-193 (brute_force_2d)
 *     origin                           pkg/src/volmoments/drt2d.py:196-208 (shift_origin)
 *   - 3D placement + cross-axis solve pkg/src/volmoments/moments3d.py:201-264
 *   - naive direct sum (Eq. 2)        pkg/src/volmoments/moments3d.py:78-139
 *                                      pkg/tests/conftest.py:40-54 (oracle_moments_3d)
 * Extension beyond the reference (documented in DESIGN.md): orders 5 and 6,
 * which add the (x+2z, y) and (x-2z, y) images (PAPER.md:98 names the
 * +-arctan(2) family; SPEC.md:152 lists it as a non-goal of the reference).
 *
 * All moment arithmetic is exact in signed __int128 (the reference uses Python
 * big ints; every supported configuration stays below 2^126, which callers
 * check with vmo_bound_ok).  Images are int64 like the reference's
 * ProjectionImage.pixels (projection.py:48-75).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef __int128 i128;

enum { VMO_XY = 0, VMO_YZ, VMO_ZX, VMO_DIAG, VMO_ANTI, VMO_X2P, VMO_X2M, VMO_NIMG };

/* number of images the DPM method needs at order K: 4 (K<=3), 5 (K=4), 6 (K=5), 7 (K=6) */
int vmo_num_images(int order) {
  if (order <= 3) return 4;
  return order + 1;
}

/* Stored image geometry (W = first index i, H = second index j; pixels[j][i])
 * and the additive offsets (ai, aj) that map stored indices to logical global
 * coordinates for a slab whose first plane is global z0 (z0 = 0: whole volume).
 * projection.py:7-14 / :189-191 for the five reference images. */
void vmo_layout(int64_t L, int64_t M, int64_t N, int64_t z0, int img,
                int64_t* W, int64_t* H, int64_t* ai, int64_t* aj) {
  switch (img) {
    case VMO_XY:   *W = L; *H = M; *ai = 0; *aj = 0; break;
    case VMO_YZ:   *W = M; *H = N; *ai = 0; *aj = z0; break;
    case VMO_ZX:   *W = N; *H = L; *ai = z0; *aj = 0; break;
    case VMO_DIAG: *W = L + N - 1; *H = M; *ai = z0; *aj = 0; break;
    case VMO_ANTI: *W = L + N - 1; *H = M; *ai = -(N - 1) - z0; *aj = 0; break;
    case VMO_X2P:  *W = L + 2 * N - 2; *H = M; *ai = 2 * z0; *aj = 0; break;
    default:       *W = L + 2 * N - 2; *H = M; *ai = -2 * (N - 1) - 2 * z0; *aj = 0; break;
  }
}

static inline int64_t voxel_at(const void* vox, int dtype, int32_t offset, size_t idx) {
  switch (dtype) {
    case 1: return ((const uint8_t*)vox)[idx];
    case 2: return ((const uint16_t*)vox)[idx];
    default: return (int64_t)((const int16_t*)vox)[idx] + offset;
  }
}

/* Single pass over the voxels (Listing 1), every image at
 * once.  imgs[k] must hold W*H int64 zeros.  Parallel over y: rows of
 * XY/DIAG/ANTI/X2P/X2M and columns of YZ are owned by one y; ZX gets
 * per-thread partials merged at the end (merge by addition). */
void vmo_project(const void* vox, int dtype, int32_t offset,
                 int64_t L, int64_t M, int64_t N, int n_img, int64_t** imgs) {
  int64_t W[VMO_NIMG], H[VMO_NIMG], ai, aj;
  for (int k = 0; k < n_img; ++k) vmo_layout(L, M, N, 0, k, &W[k], &H[k], &ai, &aj);
  int64_t* xy = imgs[VMO_XY]; int64_t* yz = imgs[VMO_YZ]; int64_t* zx = imgs[VMO_ZX];
  int64_t* dg = n_img > VMO_DIAG ? imgs[VMO_DIAG] : NULL;
  int64_t* an = n_img > VMO_ANTI ? imgs[VMO_ANTI] : NULL;
  int64_t* xp = n_img > VMO_X2P ? imgs[VMO_X2P] : NULL;
  int64_t* xm = n_img > VMO_X2M ? imgs[VMO_X2M] : NULL;
#pragma omp parallel
  {
    int64_t* zx_part = (int64_t*)calloc((size_t)(L * N), sizeof(int64_t));
#pragma omp for schedule(static)
    for (int64_t y = 0; y < M; ++y) {
      for (int64_t z = 0; z < N; ++z) {
        size_t base = (size_t)((z * M + y) * L);
        int64_t row = 0;
        for (int64_t x = 0; x < L; ++x) {
          int64_t v = voxel_at(vox, dtype, offset, base + (size_t)x);
          row += v;
          xy[y * L + x] += v;                                    /* (x, y)        */
          zx_part[x * N + z] += v;                               /* (z, x)        */
          if (dg) dg[y * W[VMO_DIAG] + x + z] += v;              /* (x+z, y)      */
          if (an) an[y * W[VMO_ANTI] + x - z + N - 1] += v;      /* (x-z+N-1, y)  */
          if (xp) xp[y * W[VMO_X2P] + x + 2 * z] += v;           /* (x+2z, y)     */
          if (xm) xm[y * W[VMO_X2M] + x - 2 * z + 2 * (N - 1)] += v;
        }
        yz[z * M + y] += row;                                    /* (y, z)        */
      }
    }
#pragma omp critical
    for (int64_t i = 0; i < L * N; ++i) zx[i] += zx_part[i];
    free(zx_part);
  }
}

static inline i128 ipow128(int64_t b, int e) {
  i128 r = 1;
  for (int k = 0; k < e; ++k) r *= b;
  return r;
}

/* Raw 2D moments M[p][q] = sum_{j,i} I[j][i] (i+ai)^p (j+aj)^q, p+q <= order,
 * written p-major: out[idx(p,q)] with idx enumerating p then q (q <= order-p).
 * Restates brute_force_2d (drt2d.py:177-193) composed with shift_origin
 * (drt2d.py:196-208): evaluating at logical coordinates is the binomial shift. */
void vmo_moments2d(const int64_t* img, int64_t W, int64_t H, int64_t ai, int64_t aj,
                   int order, i128* out) {
  int n = 0;
  for (int p = 0; p <= order; ++p)
    for (int q = 0; q <= order - p; ++q) out[n++] = 0;
  i128* rows = (i128*)calloc((size_t)(order + 1), sizeof(i128));
  for (int64_t j = 0; j < H; ++j) {
    for (int p = 0; p <= order; ++p) rows[p] = 0;
    for (int64_t i = 0; i < W; ++i) {
      int64_t v = img[j * W + i];
      if (!v) continue;
      i128 t = v;
      for (int p = 0; p <= order; ++p) { rows[p] += t; t *= (i + ai); }
    }
    n = 0;
    for (int p = 0; p <= order; ++p) {
      i128 yq = 1;
      for (int q = 0; q <= order - p; ++q) { out[n++] += rows[p] * yq; yq *= (j + aj); }
    }
  }
  free(rows);
}

static inline int idx2(int order, int p, int q) {
  /* p-major enumeration offset: sum_{p'<p} (order-p'+1) + q */
  return p * (order + 1) - p * (p - 1) / 2 + q;
}

static inline int idx3(int order, int p, int q, int r) {
  /* lexicographic (p,q,r), p+q+r <= order: moment_indices (moments3d.py:46-54) */
  int n = 0;
  for (int a = 0; a < p; ++a) { int s = order - a; n += (s + 1) * (s + 2) / 2; }
  int s = order - p;
  for (int b = 0; b < q; ++b) n += s - b + 1;
  return n + r;
}

int vmo_num_moments3d(int order) { return (order + 1) * (order + 2) * (order + 3) / 6; }
int vmo_num_moments2d(int order) { return (order + 1) * (order + 2) / 2; }

static int exact_div(i128 num, int64_t d, i128* q) {
  i128 r = num % d;
  *q = num / d;
  return r == 0;
}

static int64_t binom(int n, int k) {
  int64_t r = 1;
  for (int i = 1; i <= k; ++i) r = r * (n - k + i) / i;
  return r;
}

/* Placement (moments3d.py:223-261) + the cross-axis solve.  m2d holds
 * n_img blocks of vmo_num_moments2d(order) logical-origin 2D moments.
 * Returns 0, or a nonzero status: 1 = routes disagree (InconsistencyError
 * "disagree"), 2 = non-exact division, 3 = image masses differ.
 *
 * Cross-axis moments generalise _cross_axis_moments (moments3d.py:201-220):
 * for the (x + t z, y) image, f_t = M^t_{p,q} - M_{p,q,0} - t^p M_{0,q,p}
 * = sum_{c=1}^{p-1} C(p,c) t^c M_{p-c,q,c}, solved with t = 1,-1,2,-2.  At
 * order 4 this is exactly the reference's M111/M121/M211/M112 formulas. */
int vmo_derive3d(const i128* m2d, int order, i128* out) {
  const int n2 = vmo_num_moments2d(order);
  const int n3 = vmo_num_moments3d(order);
  const int n_img = vmo_num_images(order);
  char* have = (char*)calloc((size_t)n3, 1);
  int status = 0;
  for (int k = 1; k < n_img; ++k)
    if (m2d[k * n2 + idx2(order, 0, 0)] != m2d[idx2(order, 0, 0)]) status = 3;
#define PLACE(P, Q, R, V) do { int _i = idx3(order, P, Q, R); i128 _v = (V);          \
    if (!have[_i]) { have[_i] = 1; out[_i] = _v; }                                    \
    else if (out[_i] != _v && !status) status = 1; } while (0)
  for (int p = 0; p <= order; ++p)
    for (int q = 0; q <= order - p; ++q) PLACE(p, q, 0, m2d[0 * n2 + idx2(order, p, q)]);
  for (int p = 0; p <= order; ++p)
    for (int q = 0; q <= order - p; ++q) PLACE(0, p, q, m2d[1 * n2 + idx2(order, p, q)]);
  for (int p = 0; p <= order; ++p)
    for (int q = 0; q <= order - p; ++q) PLACE(q, 0, p, m2d[2 * n2 + idx2(order, p, q)]);
#undef PLACE
  static const int tv[4] = {1, -1, 2, -2};
  for (int q = 1; q <= order - 2; ++q) {
    for (int p = 2; p <= order - q; ++p) {
      const int n = p - 1;                       /* unknowns c = 1..p-1, images 3..3+n-1 */
      i128 f[4];
      for (int k = 0; k < n; ++k) {
        i128 tp = ipow128(tv[k], p);
        f[k] = m2d[(3 + k) * n2 + idx2(order, p, q)] - out[idx3(order, p, q, 0)]
             - tp * out[idx3(order, 0, q, p)];
      }
      i128 u[5] = {0, 0, 0, 0, 0};
      int ok = 1;
      if (n == 1) {
        u[1] = f[0];
      } else if (n == 2) {
        ok &= exact_div(f[0] + f[1], 2, &u[2]);
        ok &= exact_div(f[0] - f[1], 2, &u[1]);
      } else if (n == 3) {
        i128 S = f[0] + f[1], D = f[0] - f[1];
        ok &= exact_div(S, 2, &u[2]);
        ok &= exact_div(f[2] - 2 * S - D, 6, &u[3]);
        i128 h; ok &= exact_div(D, 2, &h); u[1] = h - u[3];
      } else {
        i128 E1, E2, O1, O2;
        ok &= exact_div(f[0] + f[1], 2, &E1); ok &= exact_div(f[2] + f[3], 2, &E2);
        ok &= exact_div(f[0] - f[1], 2, &O1); ok &= exact_div(f[2] - f[3], 2, &O2);
        ok &= exact_div(E2 - 4 * E1, 12, &u[4]); u[2] = E1 - u[4];
        ok &= exact_div(O2 - 2 * O1, 6, &u[3]); u[1] = O1 - u[3];
      }
      for (int c = 1; c <= n; ++c) {
        i128 m;
        ok &= exact_div(u[c], binom(p, c), &m);
        out[idx3(order, p - c, q, c)] = m;
        have[idx3(order, p - c, q, c)] = 1;
      }
      if (!ok && !status) status = 2;
    }
  }
  free(have);
  (void)n3;
  return status;
}

/* Whole pipeline on a volume: project -> 2D moments -> derive.  z0 shifts the
 * slab to global coordinates (the multi-GPU z-slab partial). */
int vmo_dpm(const void* vox, int dtype, int32_t offset, int64_t L, int64_t M, int64_t N,
            int64_t z0, int order, i128* out) {
  const int n_img = vmo_num_images(order);
  const int n2 = vmo_num_moments2d(order);
  int64_t* imgs[VMO_NIMG];
  int64_t W[VMO_NIMG], H[VMO_NIMG], ai[VMO_NIMG], aj[VMO_NIMG];
  for (int k = 0; k < n_img; ++k) {
    vmo_layout(L, M, N, z0, k, &W[k], &H[k], &ai[k], &aj[k]);
    imgs[k] = (int64_t*)calloc((size_t)(W[k] * H[k]), sizeof(int64_t));
  }
  vmo_project(vox, dtype, offset, L, M, N, n_img, imgs);
  i128* m2d = (i128*)calloc((size_t)(n_img * n2), sizeof(i128));
#pragma omp parallel for schedule(dynamic)
  for (int k = 0; k < n_img; ++k) vmo_moments2d(imgs[k], W[k], H[k], ai[k], aj[k], order, m2d + k * n2);
  int st = vmo_derive3d(m2d, order, out);
  for (int k = 0; k < n_img; ++k) free(imgs[k]);
  free(m2d);
  return st;
}

/* Naive direct sum, Eq. 2 (moments3d.py:78-139; conftest.py:40-54), exact:
 * M_pqr = sum V x^p y^q (z+z0)^r, factored row -> plane -> volume as in
 * factored_moments (moments3d.py:142-198).  Parallel over z with per-thread
 * partial sums (integer addition, order-independent). */
void vmo_naive(const void* vox, int dtype, int32_t offset, int64_t L, int64_t M, int64_t N,
               int64_t z0, int order, i128* out) {
  const int n3 = vmo_num_moments3d(order);
  for (int k = 0; k < n3; ++k) out[k] = 0;
#pragma omp parallel
  {
    i128* acc = (i128*)calloc((size_t)n3, sizeof(i128));
    i128* rowp = (i128*)calloc((size_t)(order + 1), sizeof(i128));
    i128* plane = (i128*)calloc((size_t)((order + 1) * (order + 1)), sizeof(i128));
#pragma omp for schedule(static)
    for (int64_t z = 0; z < N; ++z) {
      memset(plane, 0, sizeof(i128) * (size_t)((order + 1) * (order + 1)));
      for (int64_t y = 0; y < M; ++y) {
        for (int p = 0; p <= order; ++p) rowp[p] = 0;
        size_t base = (size_t)((z * M + y) * L);
        for (int64_t x = 0; x < L; ++x) {
          int64_t v = voxel_at(vox, dtype, offset, base + (size_t)x);
          if (!v) continue;
          i128 t = v;
          for (int p = 0; p <= order; ++p) { rowp[p] += t; t *= x; }
        }
        i128 yq = 1;
        for (int q = 0; q <= order; ++q) {
          for (int p = 0; p + q <= order; ++p) plane[p * (order + 1) + q] += rowp[p] * yq;
          yq *= y;
        }
      }
      i128 zr = 1;
      for (int r = 0; r <= order; ++r) {
        for (int p = 0; p + r <= order; ++p)
          for (int q = 0; p + q + r <= order; ++q)
            acc[idx3(order, p, q, r)] += plane[p * (order + 1) + q] * zr;
        zr *= (z + z0);
      }
    }
#pragma omp critical
    for (int k = 0; k < n3; ++k) out[k] += acc[k];
    free(acc); free(rowp); free(plane);
  }
}

/* The naive O(n^3)-multiply direct sum, Eq. 2, term by term: every moment
 * (p, q, r) multiplies every voxel by its own monomial x^p y^q (z+z0)^r
 * (moments3d.py:78-139 computes each (p, q, r) as a separate voxel-by-monomial
 * product before its plane and z sums).  Exact in __int128; parallel over z.
 * A CPU baseline only (bench.py), never a checker: vmo_naive is the checker. */
void vmo_naive_direct(const void* vox, int dtype, int32_t offset, int64_t L, int64_t M, int64_t N,
                      int64_t z0, int order, i128* out) {
  const int n3 = vmo_num_moments3d(order);
  int tp[128], tq[128], tr[128];
  {
    int m = 0;
    for (int p = 0; p <= order; ++p)
      for (int q = 0; p + q <= order; ++q)
        for (int r = 0; p + q + r <= order; ++r, ++m) { tp[m] = p; tq[m] = q; tr[m] = r; }
  }
  for (int k = 0; k < n3; ++k) out[k] = 0;
#pragma omp parallel
  {
    i128* acc = (i128*)calloc((size_t)n3, sizeof(i128));
    i128 px[8], py[8], pz[8];
#pragma omp for schedule(static)
    for (int64_t z = 0; z < N; ++z) {
      pz[0] = 1;
      for (int k = 1; k <= order; ++k) pz[k] = pz[k - 1] * (z + z0);
      for (int64_t y = 0; y < M; ++y) {
        py[0] = 1;
        for (int k = 1; k <= order; ++k) py[k] = py[k - 1] * y;
        const size_t base = (size_t)((z * M + y) * L);
        for (int64_t x = 0; x < L; ++x) {
          const int64_t v = voxel_at(vox, dtype, offset, base + (size_t)x);
          px[0] = 1;
          for (int k = 1; k <= order; ++k) px[k] = px[k - 1] * x;
          for (int m = 0; m < n3; ++m) acc[m] += (i128)v * px[tp[m]] * py[tq[m]] * pz[tr[m]];
        }
      }
    }
#pragma omp critical
    for (int k = 0; k < n3; ++k) out[k] += acc[k];
    free(acc);
  }
}

int vmo_max_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

void vmo_set_threads(int n) {
#ifdef _OPENMP
  if (n > 0) omp_set_num_threads(n);
#else
  (void)n;
#endif
}

/* ---- host copy of the config-5 synthetic volume generator ------------------
 * Same integer formula as paper_2012_08099_b200/csrc/synth.cu (value noise,
 * 4 octaves, quantised smoothstep weights), so CPU baselines and checks can
 * build bounded samples of the cfg5 volume without a GPU. */
static inline uint64_t vmo_mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
static inline uint64_t vmo_lattice(uint64_t seed, int o, int64_t cx, int64_t cy, int64_t cz) {
  uint64_t h = seed ^ ((uint64_t)o << 56);
  h = vmo_mix64(h ^ ((uint64_t)cx * 0x8CB92BA72F3D8DD7ull));
  h = vmo_mix64(h ^ ((uint64_t)cy * 0xA24BAED4963EE407ull));
  h = vmo_mix64(h ^ ((uint64_t)cz * 0x9FB21C651E98DF25ull));
  return h >> 48;
}
static inline uint64_t vmo_sweight(int64_t f, int64_t S) {
  return (uint64_t)((f * f * (3 * S - 2 * f)) * 65536 / (S * S * S));
}
void vmo_synth_noise_u16(uint16_t* out, int64_t L, int64_t M, int64_t z0, int64_t nz, uint64_t seed) {
  /* per row and octave the 8 lattice hashes of an x-cell are shared by its S
   * voxels: hashed once per cell, then the (bit-identical) weights per voxel */
#pragma omp parallel
  {
    uint64_t* acc = (uint64_t*)malloc((size_t)L * sizeof(uint64_t));
#pragma omp for collapse(2) schedule(static)
    for (int64_t zi = 0; zi < nz; ++zi) {
      for (int64_t y = 0; y < M; ++y) {
        const int64_t z = z0 + zi;
        for (int64_t x = 0; x < L; ++x) acc[x] = 0;
        for (int o = 0; o < 4; ++o) {
          const int64_t S = 128 >> o;
          const int64_t cy = y / S, cz = z / S;
          const uint64_t wy = vmo_sweight(y - cy * S, S), wz = vmo_sweight(z - cz * S, S);
          for (int64_t cx = 0; cx * S < L; ++cx) {
            uint64_t h[2][2][2];
            for (int dz = 0; dz < 2; ++dz)
              for (int dy = 0; dy < 2; ++dy)
                for (int dx = 0; dx < 2; ++dx) h[dz][dy][dx] = vmo_lattice(seed, o, cx + dx, cy + dy, cz + dz);
            const int64_t xe = (cx + 1) * S < L ? (cx + 1) * S : L;
            for (int64_t x = cx * S; x < xe; ++x) {
              const uint64_t wx = vmo_sweight(x - cx * S, S);
              uint64_t c[2];
              for (int dz = 0; dz < 2; ++dz) {
                const uint64_t b0 = h[dz][0][0] * (65536 - wx) + h[dz][0][1] * wx;
                const uint64_t b1 = h[dz][1][0] * (65536 - wx) + h[dz][1][1] * wx;
                c[dz] = b0 * (65536 - wy) + b1 * wy;
              }
              acc[x] += ((c[0] * (65536 - wz) + c[1] * wz) >> 48) << (3 - o);
            }
          }
        }
        for (int64_t x = 0; x < L; ++x) out[(zi * M + y) * L + x] = (uint16_t)(acc[x] / 15);
      }
    }
    free(acc);
  }
}
