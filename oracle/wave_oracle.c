/*
 * TEST INFRASTRUCTURE ONLY — CPU oracle for the superposed-adjoint hot path.
 *
 * Plain-C restatement of the reference's Numba inner loops
 * (/root/reference/pkg/src/waveopt/kernels.py).  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * may load this library; the product path (paper_2509_15744_b200) never does.
 *
 * Arithmetic contract: every expression keeps the reference's evaluation
 * order and rounding (IEEE-754 binary32/binary64, round-to-nearest, no FMA
 * contraction, no flush-to-zero).  Build with -ffp-contract=off and without
 * -ffast-math (oracle/Makefile).  The outer axis-0 loop is split across
 * OpenMP threads; every cell is computed independently, so the result is
 * bitwise independent of the thread count.
 *
 * Parity is pinned against the reference itself: tests/golden/ fixtures were
 * produced by tests/golden/make_golden.py running waveopt from
 * /root/reference, and tests/test_oracle_golden.py checks this file against
 * them bit for bit.
 */
#include <stdint.h>
#include <stddef.h>

#define IDX3(i, j, k) (((int64_t)(i) * n1 + (j)) * n2 + (k))
#define IDX2(i, j) ((int64_t)(i) * n1 + (j))

/* ------------------------------------------------------------------ */
/* Stencil: kernels.py:18-69 (step_1d / step_2d / step_3d).           */
/* acc = u - u; per axis in order 0,1,2:                               */
/*   if i < n-1: acc += (u[i+1]-u[i]) * wf[i]                          */
/*   if i > 0:   acc -= (u[i]-u[i-1]) * wf[i-1]                        */
/* out = ((u + u) - u_prev) + coef * acc                               */
/* ------------------------------------------------------------------ */
#define DEFINE_STEP(T, SUF)                                                        \
static void step_1d_##SUF(int64_t n0, const T *u_prev, const T *u, const T *wf0,  \
                          const T *coef, T *out) {                                 \
    _Pragma("omp parallel for schedule(static)")                                   \
    for (int64_t i = 0; i < n0; ++i) {                                             \
        T acc = u[i] - u[i];                                                       \
        if (i < n0 - 1) acc += (u[i + 1] - u[i]) * wf0[i];                         \
        if (i > 0) acc -= (u[i] - u[i - 1]) * wf0[i - 1];                          \
        out[i] = u[i] + u[i] - u_prev[i] + coef[i] * acc;                          \
    }                                                                              \
}                                                                                  \
static void step_2d_##SUF(int64_t n0, int64_t n1, const T *u_prev, const T *u,    \
                          const T *wf0, const T *wf1, const T *coef, T *out) {     \
    /* wf0 has shape (n0-1, n1); wf1 has shape (n0, n1-1) */                       \
    _Pragma("omp parallel for schedule(static)")                                   \
    for (int64_t i = 0; i < n0; ++i) {                                             \
        for (int64_t j = 0; j < n1; ++j) {                                         \
            const int64_t c = IDX2(i, j);                                          \
            T acc = u[c] - u[c];                                                   \
            if (i < n0 - 1) acc += (u[IDX2(i + 1, j)] - u[c]) * wf0[IDX2(i, j)];   \
            if (i > 0) acc -= (u[c] - u[IDX2(i - 1, j)]) * wf0[IDX2(i - 1, j)];    \
            if (j < n1 - 1) acc += (u[c + 1] - u[c]) * wf1[i * (n1 - 1) + j];      \
            if (j > 0) acc -= (u[c] - u[c - 1]) * wf1[i * (n1 - 1) + j - 1];       \
            out[c] = u[c] + u[c] - u_prev[c] + coef[c] * acc;                      \
        }                                                                          \
    }                                                                              \
}                                                                                  \
static void step_3d_##SUF(int64_t n0, int64_t n1, int64_t n2, const T *u_prev,    \
                          const T *u, const T *wf0, const T *wf1, const T *wf2,    \
                          const T *coef, T *out) {                                 \
    /* wf0: (n0-1,n1,n2)  wf1: (n0,n1-1,n2)  wf2: (n0,n1,n2-1) */                  \
    _Pragma("omp parallel for schedule(static)")                                   \
    for (int64_t i = 0; i < n0; ++i) {                                             \
        for (int64_t j = 0; j < n1; ++j) {                                         \
            for (int64_t k = 0; k < n2; ++k) {                                     \
                const int64_t c = IDX3(i, j, k);                                   \
                T acc = u[c] - u[c];                                               \
                if (i < n0 - 1)                                                    \
                    acc += (u[IDX3(i + 1, j, k)] - u[c]) * wf0[c];                 \
                if (i > 0)                                                         \
                    acc -= (u[c] - u[IDX3(i - 1, j, k)]) * wf0[IDX3(i - 1, j, k)]; \
                const int64_t c1 = ((int64_t)i * (n1 - 1) + j) * n2 + k;           \
                if (j < n1 - 1) acc += (u[IDX3(i, j + 1, k)] - u[c]) * wf1[c1];    \
                if (j > 0)                                                         \
                    acc -= (u[c] - u[IDX3(i, j - 1, k)]) * wf1[c1 - n2];           \
                const int64_t c2 = ((int64_t)i * n1 + j) * (n2 - 1) + k;           \
                if (k < n2 - 1) acc += (u[c + 1] - u[c]) * wf2[c2];                \
                if (k > 0) acc -= (u[c] - u[c - 1]) * wf2[c2 - 1];                 \
                out[c] = u[c] + u[c] - u_prev[c] + coef[c] * acc;                  \
            }                                                                      \
        }                                                                          \
    }                                                                              \
}

DEFINE_STEP(float, f32)
DEFINE_STEP(double, f64)

/* ------------------------------------------------------------------ */
/* Kernel increment: kernels.py:72-128.                                */
/* va = (a_new-a_old)*inv2dt ; g = (a_mid[ip]-a_mid[im])*inv2dx        */
/* (clamped ip/im); acc += sdt*(cv*va*vb + cg*(ga0*gb0 + ga1*gb1 + ..)) */
/* ------------------------------------------------------------------ */
#define DEFINE_KI(T, SUF)                                                          \
static void ki_1d_##SUF(int64_t n0, T *acc, const T *ao, const T *am, const T *an,\
                        const T *bo, const T *bm, const T *bn, T cv, T cg,         \
                        T inv2dt, T inv2dx, T sdt) {                               \
    _Pragma("omp parallel for schedule(static)")                                   \
    for (int64_t i = 0; i < n0; ++i) {                                             \
        int64_t im = i > 0 ? i - 1 : 0, ip = i < n0 - 1 ? i + 1 : n0 - 1;          \
        T va = (an[i] - ao[i]) * inv2dt;                                           \
        T vb = (bn[i] - bo[i]) * inv2dt;                                           \
        T ga = (am[ip] - am[im]) * inv2dx;                                         \
        T gb = (bm[ip] - bm[im]) * inv2dx;                                         \
        acc[i] += sdt * (cv * va * vb + cg * ga * gb);                             \
    }                                                                              \
}                                                                                  \
static void ki_2d_##SUF(int64_t n0, int64_t n1, T *acc, const T *ao, const T *am, \
                        const T *an, const T *bo, const T *bm, const T *bn, T cv,  \
                        T cg, T inv2dt, T inv2dx, T sdt) {                         \
    _Pragma("omp parallel for schedule(static)")                                   \
    for (int64_t i = 0; i < n0; ++i) {                                             \
        int64_t im = i > 0 ? i - 1 : 0, ip = i < n0 - 1 ? i + 1 : n0 - 1;          \
        for (int64_t j = 0; j < n1; ++j) {                                         \
            int64_t jm = j > 0 ? j - 1 : 0, jp = j < n1 - 1 ? j + 1 : n1 - 1;      \
            const int64_t c = IDX2(i, j);                                          \
            T va = (an[c] - ao[c]) * inv2dt;                                       \
            T vb = (bn[c] - bo[c]) * inv2dt;                                       \
            T ga0 = (am[IDX2(ip, j)] - am[IDX2(im, j)]) * inv2dx;                  \
            T gb0 = (bm[IDX2(ip, j)] - bm[IDX2(im, j)]) * inv2dx;                  \
            T ga1 = (am[IDX2(i, jp)] - am[IDX2(i, jm)]) * inv2dx;                  \
            T gb1 = (bm[IDX2(i, jp)] - bm[IDX2(i, jm)]) * inv2dx;                  \
            acc[c] += sdt * (cv * va * vb + cg * (ga0 * gb0 + ga1 * gb1));         \
        }                                                                          \
    }                                                                              \
}                                                                                  \
static void ki_3d_##SUF(int64_t n0, int64_t n1, int64_t n2, T *acc, const T *ao,  \
                        const T *am, const T *an, const T *bo, const T *bm,        \
                        const T *bn, T cv, T cg, T inv2dt, T inv2dx, T sdt) {      \
    _Pragma("omp parallel for schedule(static)")                                   \
    for (int64_t i = 0; i < n0; ++i) {                                             \
        int64_t im = i > 0 ? i - 1 : 0, ip = i < n0 - 1 ? i + 1 : n0 - 1;          \
        for (int64_t j = 0; j < n1; ++j) {                                         \
            int64_t jm = j > 0 ? j - 1 : 0, jp = j < n1 - 1 ? j + 1 : n1 - 1;      \
            for (int64_t k = 0; k < n2; ++k) {                                     \
                int64_t km = k > 0 ? k - 1 : 0, kp = k < n2 - 1 ? k + 1 : n2 - 1;  \
                const int64_t c = IDX3(i, j, k);                                   \
                T va = (an[c] - ao[c]) * inv2dt;                                   \
                T vb = (bn[c] - bo[c]) * inv2dt;                                   \
                T ga0 = (am[IDX3(ip, j, k)] - am[IDX3(im, j, k)]) * inv2dx;        \
                T gb0 = (bm[IDX3(ip, j, k)] - bm[IDX3(im, j, k)]) * inv2dx;        \
                T ga1 = (am[IDX3(i, jp, k)] - am[IDX3(i, jm, k)]) * inv2dx;        \
                T gb1 = (bm[IDX3(i, jp, k)] - bm[IDX3(i, jm, k)]) * inv2dx;        \
                T ga2 = (am[IDX3(i, j, kp)] - am[IDX3(i, j, km)]) * inv2dx;        \
                T gb2 = (bm[IDX3(i, j, kp)] - bm[IDX3(i, j, km)]) * inv2dx;        \
                acc[c] += sdt * (cv * va * vb                                      \
                                 + cg * (ga0 * gb0 + ga1 * gb1 + ga2 * gb2));      \
            }                                                                      \
        }                                                                          \
    }                                                                              \
}

DEFINE_KI(float, f32)
DEFINE_KI(double, f64)

/* ------------------------------------------------------------------ */
/* ctypes entry points (oracle/oracle.py)                              */
/* ------------------------------------------------------------------ */

/* kernels.py:136-139 apply_step; wf[a] may be NULL for a >= ndim */
int or_apply_step(int itemsize, int ndim, const int64_t *shape, const void *u_prev,
                  const void *u_cur, const void *wf0, const void *wf1, const void *wf2,
                  const void *coef, void *out) {
    if (itemsize == 4) {
        if (ndim == 1) step_1d_f32(shape[0], u_prev, u_cur, wf0, coef, out);
        else if (ndim == 2) step_2d_f32(shape[0], shape[1], u_prev, u_cur, wf0, wf1, coef, out);
        else if (ndim == 3)
            step_3d_f32(shape[0], shape[1], shape[2], u_prev, u_cur, wf0, wf1, wf2, coef, out);
        else return 1;
    } else if (itemsize == 8) {
        if (ndim == 1) step_1d_f64(shape[0], u_prev, u_cur, wf0, coef, out);
        else if (ndim == 2) step_2d_f64(shape[0], shape[1], u_prev, u_cur, wf0, wf1, coef, out);
        else if (ndim == 3)
            step_3d_f64(shape[0], shape[1], shape[2], u_prev, u_cur, wf0, wf1, wf2, coef, out);
        else return 1;
    } else return 1;
    return 0;
}

/* kernels.py:142-152 apply_kernel_increment; the five scalars arrive as the
 * fp64 values the reference computes and are cast to the accumulator dtype
 * here, exactly like `dt_(cv)` at kernels.py:149-152. */
int or_apply_kernel_increment(int itemsize, int ndim, const int64_t *shape, void *acc,
                              const void *ao, const void *am, const void *an,
                              const void *bo, const void *bm, const void *bn,
                              double cv, double cg, double inv2dt, double inv2dx,
                              double sdt) {
    if (itemsize == 4) {
        float fcv = (float)cv, fcg = (float)cg, fi2t = (float)inv2dt, fi2x = (float)inv2dx,
              fsdt = (float)sdt;
        if (ndim == 1) ki_1d_f32(shape[0], acc, ao, am, an, bo, bm, bn, fcv, fcg, fi2t, fi2x, fsdt);
        else if (ndim == 2)
            ki_2d_f32(shape[0], shape[1], acc, ao, am, an, bo, bm, bn, fcv, fcg, fi2t, fi2x, fsdt);
        else if (ndim == 3)
            ki_3d_f32(shape[0], shape[1], shape[2], acc, ao, am, an, bo, bm, bn, fcv, fcg, fi2t,
                      fi2x, fsdt);
        else return 1;
    } else if (itemsize == 8) {
        if (ndim == 1) ki_1d_f64(shape[0], acc, ao, am, an, bo, bm, bn, cv, cg, inv2dt, inv2dx, sdt);
        else if (ndim == 2)
            ki_2d_f64(shape[0], shape[1], acc, ao, am, an, bo, bm, bn, cv, cg, inv2dt, inv2dx, sdt);
        else if (ndim == 3)
            ki_3d_f64(shape[0], shape[1], shape[2], acc, ao, am, an, bo, bm, bn, cv, cg, inv2dt,
                      inv2dx, sdt);
        else return 1;
    } else return 1;
    return 0;
}

/* solver.py:180-186 check_finite: max |u| (the comparison happens in Python) */
double or_max_abs(int itemsize, int64_t n, const void *u) {
    double m = 0.0;
    if (itemsize == 4) {
        const float *p = u;
        float mf = 0.0f;
        for (int64_t i = 0; i < n; ++i) {
            float a = p[i] < 0 ? -p[i] : p[i];
            if (a != a) return a; /* NaN */
            if (a > mf) mf = a;
        }
        m = mf;
    } else {
        const double *p = u;
        for (int64_t i = 0; i < n; ++i) {
            double a = p[i] < 0 ? -p[i] : p[i];
            if (a != a) return a;
            if (a > m) m = a;
        }
    }
    return m;
}

int or_num_threads(void) {
#ifdef _OPENMP
    extern int omp_get_max_threads(void);
    return omp_get_max_threads();
#else
    return 1;
#endif
}
