/*
 * phantom/phantom.c -- seeded synthetic chest-CT phantom with an airway tube
 * tree.  This is the ONE input generator shared by the CUDA path's tests/bench
 * and the oracle; it holds none of the method's arithmetic (no histogram, no
 * entropy, no thresholds) -- it only writes voxel values.
 *
 * Recipe:
 *   HU per voxel, geometry in pixel units scaled by s = nx / 512:
 *     outside the circular field of view (radius nx/2)      -2000
 *     air inside the FOV                                    -1000
 *     body ellipse (soft tissue)                              +40
 *     subcutaneous fat ring (outer 10 % of the body)         -100
 *     two lung ellipsoids                                    -850
 *     spine + ribs                                           +700
 *     airway tree: trachea (r = 13 s px) from the top slice to a carina at
 *       40 % depth, then recursive bifurcation, child radius r * 2^(-1/3)
 *       (Murray), +-35 deg, segment length 3 r, 8 generations; lumen -1000,
 *       wall (0.3 r thick) -50.
 *   noise: integer Irwin-Hall: sum of four bytes of splitmix64(seed, z, y, x),
 *     centred and scaled by 173/1024 (sigma ~ 25 HU); none outside the FOV.
 *   output: u8  = clamp((HU + 1024) >> 3, 0, 255)      (8-bit window, R12)
 *           u16 = clamp(HU + 1024, 0, 4095)            (12-bit, R13)
 *           i16 = HU itself (dtype code 3; background -2000 exactly)
 * Geometry uses fp64 on the host; the same bytes feed GPU and oracle.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
  double x0, y0, z0, x1, y1, z1, r;
} seg_t;

static uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

/* Build the airway tree in (x, y, z) with x,y in pixels relative to the image
 * centre and z in slice units.  Returns the number of segments. */
static int build_tree(seg_t *segs, int cap, double s, double depth, double dz_per_px) {
  int n = 0;
  double r0 = 13.0 * s;
  double zc = 0.4 * depth;
  /* trachea: vertical, slightly anterior of centre */
  double tx = 0.0, ty = -0.08 * 256.0 * s;
  segs[n++] = (seg_t){tx, ty, -1.0, tx, ty, zc, r0};
  /* recursive bifurcation, breadth first */
  typedef struct {
    double x, y, z, dx, dy, dz, r;
    double px, py, pz; /* branching plane normal helper */
    int gen;
  } node_t;
  node_t *stack = (node_t *)malloc(sizeof(node_t) * 4096);
  int top = 0;
  stack[top++] = (node_t){tx, ty, zc, 0.0, 0.0, 1.0, r0, 1.0, 0.0, 0.0, 0};
  const double ang = 35.0 * M_PI / 180.0;
  while (top > 0) {
    node_t nd = stack[--top];
    if (nd.gen >= 8) continue;
    double rc = nd.r * pow(2.0, -1.0 / 3.0);
    if (rc < 0.75) continue;
    /* rotate direction by +-ang in the plane spanned by d and p */
    double dxp = nd.px, dyp = nd.py, dzp = nd.pz;
    for (int side = -1; side <= 1; side += 2) {
      double ca = cos(ang), sa = sin(ang) * side;
      double ex = ca * nd.dx + sa * dxp, ey = ca * nd.dy + sa * dyp, ez = ca * nd.dz + sa * dzp;
      double en = sqrt(ex * ex + ey * ey + ez * ez);
      ex /= en; ey /= en; ez /= en;
      if (ez < 0.15) { /* keep the tree descending */
        ez = 0.15;
        en = sqrt(ex * ex + ey * ey + ez * ez);
        ex /= en; ey /= en; ez /= en;
      }
      double len = 3.0 * rc * (nd.gen == 0 ? 2.0 : 1.0);
      double x1 = nd.x + ex * len, y1 = nd.y + ey * len, z1 = nd.z + ez * len * dz_per_px;
      if (n < cap) segs[n++] = (seg_t){nd.x, nd.y, nd.z, x1, y1, z1, rc};
      /* next plane: perpendicular to the current one (cross of e and old p) */
      double qx = ey * dzp - ez * dyp, qy = ez * dxp - ex * dzp, qz = ex * dyp - ey * dxp;
      double qn = sqrt(qx * qx + qy * qy + qz * qz);
      if (qn < 1e-9) { qx = 0; qy = 1; qz = 0; qn = 1; }
      if (top < 4096)
        stack[top++] = (node_t){x1, y1, z1, ex, ey, ez, rc, qx / qn, qy / qn, qz / qn, nd.gen + 1};
    }
  }
  free(stack);
  return n;
}

static inline int inside_ellipse(double x, double y, double cx, double cy, double ax, double ay) {
  double u = (x - cx) / ax, v = (y - cy) / ay;
  return u * u + v * v <= 1.0;
}

/* Generate slices [z_first, z_first + nz) of a phantom that is z_total slices
 * deep.  out: [nz][ny][nx] u8 (dtype_bytes 1) or u16 (2).  Deterministic in
 * (seed, nx, ny, z_total, absolute z, y, x) and independent of nthreads. */
int phantom_generate(void *out, int dtype_bytes, int64_t nx, int64_t ny, int64_t nz,
                     int64_t z_first, int64_t z_total, uint64_t seed, int nthreads) {
  if (nx <= 0 || ny <= 0 || nz <= 0 || z_total <= 0) return 1;
  double s = (double)nx / 512.0;
  double cx = 0.5 * (double)nx, cy = 0.5 * (double)ny;
  double fov_r = 0.5 * (double)nx;
  double dz_per_px = 0.7 / 1.0; /* 0.7 mm pixels, 1 mm slices */
  seg_t *segs = (seg_t *)malloc(sizeof(seg_t) * 4096);
  int nseg = build_tree(segs, 4096, s, (double)z_total, dz_per_px);
  if (nthreads < 1) nthreads = 1;
#pragma omp parallel for schedule(dynamic, 1) num_threads(nthreads)
  for (int64_t zi = 0; zi < nz; zi++) {
    int64_t z = z_first + zi;
    double zf = (double)z;
    double depth = zf / (double)z_total; /* 0 top .. 1 bottom */
    int16_t *hu = (int16_t *)malloc(sizeof(int16_t) * nx * ny);
    /* lung size grows towards mid depth */
    double lung_scale = 0.55 + 0.45 * sin(M_PI * fmin(1.0, depth * 1.2));
    for (int64_t y = 0; y < ny; y++) {
      for (int64_t x = 0; x < nx; x++) {
        double px = (double)x + 0.5 - cx, py = (double)y + 0.5 - cy;
        int v;
        if (px * px + py * py > fov_r * fov_r) {
          v = -2000;
        } else {
          v = -1000;
          double bax = 0.44 * nx, bay = 0.32 * ny;
          if (inside_ellipse(px, py, 0, 0.02 * ny, bax, bay)) {
            v = -100; /* fat ring */
            if (inside_ellipse(px, py, 0, 0.02 * ny, 0.9 * bax, 0.88 * bay)) v = 40;
            /* lungs */
            double lax = 0.15 * nx * lung_scale, lay = 0.21 * ny * lung_scale;
            if (inside_ellipse(px, py, -0.19 * nx, -0.01 * ny, lax, lay) ||
                inside_ellipse(px, py, 0.19 * nx, -0.01 * ny, lax, lay))
              v = -850;
            /* spine */
            if (inside_ellipse(px, py, 0, 0.22 * ny, 0.05 * nx, 0.05 * ny)) v = 700;
            /* ribs: 10 small discs on an ellipse just inside the fat ring */
            for (int rb = 0; rb < 10; rb++) {
              double th = M_PI * (0.15 + 0.7 * rb / 9.0);
              double rx = 0.8 * bax * cos(th);
              double ry = 0.02 * ny + 0.8 * bay * sin(th) * (rb % 2 ? 1 : -1);
              if (inside_ellipse(px, py, rx, ry, 0.018 * nx, 0.018 * nx)) v = 700;
            }
          }
        }
        hu[y * nx + x] = (int16_t)v;
      }
    }
    /* airway tree: every segment crossing the slab [z-0.5, z+0.5] */
    for (int si = 0; si < nseg; si++) {
      seg_t g = segs[si];
      double zlo = fmin(g.z0, g.z1), zhi = fmax(g.z0, g.z1);
      if (zhi < zf - 0.5 || zlo > zf + 0.5) continue;
      double dx = g.x1 - g.x0, dy = g.y1 - g.y0, dzs = g.z1 - g.z0;
      double L = sqrt(dx * dx + dy * dy);
      int steps = (int)(L / 0.5) + 1;
      double rw = g.r * 1.3;
      for (int st = 0; st <= steps; st++) {
        double u = (double)st / (double)steps;
        double zs = g.z0 + u * dzs;
        if (fabs(zs - zf) > 0.5 && steps > 1) continue;
        double sx = g.x0 + u * dx + cx, sy = g.y0 + u * dy + cy;
        int64_t xa = (int64_t)floor(sx - rw - 1), xb = (int64_t)ceil(sx + rw + 1);
        int64_t ya = (int64_t)floor(sy - rw - 1), yb = (int64_t)ceil(sy + rw + 1);
        if (xa < 0) xa = 0;
        if (ya < 0) ya = 0;
        if (xb > nx - 1) xb = nx - 1;
        if (yb > ny - 1) yb = ny - 1;
        for (int64_t y = ya; y <= yb; y++)
          for (int64_t x = xa; x <= xb; x++) {
            double ex = (double)x + 0.5 - sx, ey = (double)y + 0.5 - sy;
            double d2 = ex * ex + ey * ey;
            int16_t *h = &hu[y * nx + x];
            if (*h == -2000) continue;
            if (d2 <= g.r * g.r)
              *h = -1000 + 1; /* lumen marker (odd) -> -1000 below */
            else if (d2 <= rw * rw && *h != -999)
              *h = -50;
          }
      }
    }
    /* noise + window */
    for (int64_t y = 0; y < ny; y++) {
      for (int64_t x = 0; x < nx; x++) {
        int v = hu[y * nx + x];
        if (v == -999) v = -1000;
        if (v != -2000) {
          uint64_t key = seed ^ splitmix64((uint64_t)z * 0x100000001B3ull ^
                                           splitmix64(((uint64_t)y << 32) | (uint64_t)x));
          uint64_t hsh = splitmix64(key);
          int ih = (int)(hsh & 0xff) + (int)((hsh >> 8) & 0xff) + (int)((hsh >> 16) & 0xff) +
                   (int)((hsh >> 24) & 0xff);
          int noise = ((ih - 510) * 173) >> 10; /* arithmetic shift: floor */
          v += noise;
        }
        int64_t o = (zi * ny + y) * nx + x;
        if (dtype_bytes == 3) { /* raw int16 HU (pre-processing input) */
          ((int16_t *)out)[o] = (int16_t)v;
        } else if (dtype_bytes == 1) {
          int w = (v + 1024) >> 3;
          if (w < 0) w = 0;
          if (w > 255) w = 255;
          ((uint8_t *)out)[o] = (uint8_t)w;
        } else {
          int w = v + 1024;
          if (w < 0) w = 0;
          if (w > 4095) w = 4095;
          ((uint16_t *)out)[o] = (uint16_t)w;
        }
      }
    }
    free(hu);
  }
  free(segs);
  return 0;
}
