/*
 * hermb200 — C ABI of the B200-native Hermite wave-solver hot path.
 *
 * The reference package (`hermwave`, pure Python/numpy) has no FFI: its
 * boundary is the Python functions re-exported in pkg/src/hermwave/__init__.py.
 * Each entry point below replaces one of them; the Python mirror in
 * paper_1802_05246_b200/ binds these symbols with ctypes.
 *
 * Conventions
 *  - All field pointers are DEVICE pointers (FP64, C order), laid out exactly
 *    like the reference's Field arrays:
 *        2D  values[i][j][k][l]  (grid.py:113-116; k = x order, l = y order)
 *        1D  values[i][l]        (grid.py:82-84)
 *  - Every call is stream-ordered on `stream` (a cudaStream_t; NULL = legacy
 *    default stream) and returns an int status: 0 ok, < 0 error.  The error
 *    text is available from hw_last_error() (thread local).  No call throws.
 *  - Scalars (dt, h, speed) are passed exactly as the reference computes them
 *    (SchemeConfig.dt, Grid.h), so a caller reproduces the reference's
 *    time bookkeeping on the host.
 */
#ifndef HERMB200_H
#define HERMB200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* boundary.py:24 KINDS */
#define HW_PERIODIC   0
#define HW_DIRICHLET0 1
#define HW_NEUMANN0   2

/* grid.py:19-20 PRIMAL / DUAL */
#define HW_PRIMAL 0
#define HW_DUAL   1

#define HW_OK            0
#define HW_EINVAL       -1
#define HW_ECUDA        -2
#define HW_EUNSUPPORTED -3

/* One axis of BoundarySpec (boundary.py:29-47). */
typedef struct {
  int32_t left_kind, right_kind;
  double left_value, right_value;
} hw_axis_bc;

/*
 * Source-row view of a 2D field for one half step, with optional slab
 * decomposition along x (axis 0).  Rows [row0, row0+nrows) are local and
 * contiguous at `base`; `halo_lo` / `halo_hi` (may be NULL) hold global rows
 * row0-1 / row0+nrows received from the neighbouring ranks.  On a single
 * device: row0 = 0, nrows = nx, halos NULL.
 */
typedef struct {
  const double* base;
  const double* halo_lo;
  const double* halo_hi;
  int64_t row0, nrows;
} hw_rows2d;

/* Common 2D step geometry (grid.py:58-79, boundary.py:101-168). */
typedef struct {
  int64_t nx, ny;          /* GLOBAL source node counts of the source parity */
  int32_t parity_src;      /* HW_PRIMAL / HW_DUAL */
  int32_t periodic;        /* Grid2D.periodic */
  hw_axis_bc bcx, bcy;     /* BoundarySpec2D.x / .y (values used for u only) */
  int64_t trow0, ntrows;   /* target rows to produce (global index, count);
                              ntrows < 0 => all target rows */
} hw_geom2d;

/* Library info. */
const char* hw_last_error(void);
int hw_version(void);              /* 4: + hw_inner2d (2D conservative energy) */
int hw_max_order(void);            /* largest m with a compiled fast path */

/* interp.py:51-75 interp_matrix(mu): (2mu+2)^2 row-major, exact doubles. */
int hw_interp_matrix(int mu, double* out_host);

/*
 * Per-cell linear map of a 2D step (host only; used to pin the kernels'
 * operator against the reference on the CPU).  scheme: 0 = half_step_2d
 * (dissipative.py:215-247), 1 = full_step_conservative without the
 * `- previous` term (conservative.py:130-136), 2 = bootstrap_first_half
 * (conservative.py:185-195).  hw_cell_map_dims gives din (inputs per corner
 * node) and dout (outputs per target node); hw_cell_map_2d writes the dense
 * dout x (4 din) matrix, column = corner * din + e with corner = 2 sx + sy
 * (sx, sy = 1 for the right / upper neighbour) and e running over the first
 * input field's (k, l) entries, then the second's.
 */
int hw_cell_map_dims(int scheme, int m, int* din, int* dout);
int hw_cell_map_2d(int scheme, int m, double dt, double hx, double hy, double speed, int stages,
                   double* out_host);

/* Number of target nodes per axis produced from `n_src` source nodes. */
int64_t hw_target_count(int64_t n_src, int parity_src, int periodic);

/*
 * The three 2D steps accept every order the reference does, m = 1..12
 * (interp.py:30, 62-63; larger m -> HW_EINVAL).  The operator is the per-class
 * cell map above; which kernel applies it is an implementation detail
 * (tensor-core DMMA cell map, the SIMT constant-operand cell map, or the
 * generic runtime-order kernel above m = 8) and does not change the ABI.
 */

/*
 * dissipative.py:215-247 half_step_2d (stabilised 2D half step).
 * u: orders (m,m), v: orders (m-1,m-1).  Writes target rows
 * [trow0, trow0+ntrows) of the opposite parity into u_dst / v_dst
 * (row trow0 at offset 0).  stage_cap <= 0 selects the default 4m+4.
 */
int hw_diss2d_half_step(const hw_rows2d* u_src, const hw_rows2d* v_src,
                        double* u_dst, double* v_dst, int m,
                        const hw_geom2d* geom, double dt, double hx, double hy,
                        double speed, int stage_cap, void* stream);

/*
 * conservative.py:139-157 full_step_conservative (2D):
 * out = 2 * WT . I_{m,m}(current) - previous.  `out` may alias `previous`.
 */
int hw_cons2d_step(const hw_rows2d* cur_src, const double* prev, double* out,
                   int m, const hw_geom2d* geom, double dt, double hx, double hy,
                   double speed, void* stream);

/*
 * conservative.py:166-195 bootstrap_first_half (2D): plain recursion on
 * I_m g0 and I_m g1 (both order (m,m)), 4m+4 stages, evaluated at theta=1/2.
 */
int hw_boot2d(const hw_rows2d* g0_src, const hw_rows2d* g1_src, double* out,
              int m, const hw_geom2d* geom, double dt, double hx, double hy,
              double speed, void* stream);

/*
 * dissipative.py:160-181 half_step_1d.  forcing (may be NULL) is a device
 * array F[s-1][l][t] (s = 1..stages, l < 2m, t < n_targets) of the already
 * scaled terms h^l dt^s/(l! s!) f(l, s-1, x_t, time) (dissipative.py:102-105).
 */
int hw_diss1d_half_step(const double* u_src, const double* v_src,
                        double* u_dst, double* v_dst, int m, int64_t n_src,
                        int parity_src, const hw_axis_bc* bc, double dt,
                        double h, double speed, int stages,
                        const double* forcing, void* stream);

/* conservative.py:139-157 full_step_conservative (1D).  out may alias prev. */
int hw_cons1d_step(const double* cur, const double* prev, double* out, int m,
                   int64_t n_src, int parity_src, const hw_axis_bc* bc,
                   double lam, void* stream);

/* conservative.py:166-184 bootstrap_first_half (1D), 2m+3 stages. */
int hw_boot1d(const double* g0, const double* g1, double* out, int m,
              int64_t n_src, int parity_src, const hw_axis_bc* bc, double dt,
              double h, double speed, void* stream);

/*
 * diagnostics.py:118-135 l2_error_field_2d, reduced on the device.
 * The field (orders (mx,my)) is interpolated on every target cell of its own
 * corner gather and evaluated at npts^2 Gauss points; `exact` is either a
 * device array exact[ci][cj][p][q] (exact_kind = 0) or one of the built-in
 * closed forms (exact_kind = 1 plane wave sin(w(x+y+sqrt2 t)), params =
 * {w, t}; exact_kind = 2 standing wave sin(kx x) sin(ky y) cos(om t),
 * params = {kx, ky, om, t}).  Node coordinates: x_left/y_left, hx/hy.
 * Result (the sum before sqrt, i.e. the squared error) is written to
 * *out_host after a stream synchronisation.
 */
int hw_l2err2d(const hw_rows2d* src, int mx, int my, const hw_geom2d* geom,
               double x_left, double y_left, double hx, double hy, int npts,
               const double* gauss_x, const double* gauss_w,
               int exact_kind, const double* exact, const double* params,
               double* out_host, void* stream);

/*
 * Squared 2D seminorm sum_cells int int (d^dx/dx^dx d^dy/dy^dy I u)^2 dx dy
 * of the tensor interpolant I = I_{mx,my} over the target cells of the
 * field's own corner gather (the cells of hw_l2err2d), by npts^2-point Gauss
 * quadrature (exact when 2 npts - 1 >= 2 (2 max(mx,my) + 1)).  The building
 * block of the defined 2D energy (norms.py dissipative_energy_2d; no
 * reference counterpart: diagnostics.py:220-234 is 1D only).  Result ->
 * *out_host after a stream synchronisation.
 */
int hw_seminorm2d(const hw_rows2d* src, int mx, int my, const hw_geom2d* geom,
                  double hx, double hy, int dx, int dy, int npts,
                  const double* gauss_x, const double* gauss_w,
                  double* out_host, void* stream);

/*
 * Bilinear 2D seminorm: sum over the target cells [trow0, trow0+ntrows) of
 * the field's corner gather of w_cell * int int (D I f)(D I g) dx dy, with
 * D = d^dx/dx^dx d^dy/dy^dy and I = I_{mx,my} the tensor interpolant, by
 * npts^2-point Gauss quadrature (exact for 2 npts - 1 >= 2 (2 m + 1) - dx - dy
 * per axis).  g = NULL means g = f.  wall_half != 0: a cell whose gather used
 * a wall ghost (dual parity on a wall grid) straddles the wall and counts
 * 1/2 per such axis, i.e. the integral over the physical domain of the
 * reflected extension the ghosts define (boundary.py:56-98).  Accumulated in
 * double-double.  The building block of the 2D conservative energy
 * (norms.py conservative_energy_2d; the reference's conservative_energy,
 * diagnostics.py:190-226, is 1D and periodic only).  Slabs: pass a row window
 * with halos and sum the per-rank results.  -> *out_host after a stream sync.
 */
int hw_inner2d(const hw_rows2d* f, const hw_rows2d* g, int mx, int my, const hw_geom2d* geom,
               double hx, double hy, int dx, int dy, int npts,
               const double* gauss_x, const double* gauss_w, int wall_half,
               double* out_host, void* stream);

/*
 * diagnostics.py:66-115 per-piece 1D L2 errors.  For each target piece t the
 * caller supplies the clipped Gauss abscissae in the piece's scaled variable
 * (xi[t][p]), the weights times half-width (w[t][p]) and the exact values
 * ex[t][p]; deriv selects the field (0) or its first derivative (1, scaled
 * by 1/h like CellPolynomial.derivative).  Squared error -> *out_host.
 */
int hw_l2err1d(const double* src, int mu, int64_t n_src, int parity_src,
               const hw_axis_bc* bc, double h, int deriv, int npts,
               const double* xi, const double* w, const double* ex,
               double* out_host, void* stream);

/*
 * diagnostics.py:201-212 seminorm_sq of the global interpolant of a 1D field
 * (pieces = cells of the field's own gather, ghosts with the bc's values as
 * field_interpolant does): scale * sum over pieces of the Gauss integral
 * (npts points, nodes gx / weights gw on [-1, 1], host pointers) of the squared
 * order-th derivative.  dissipative_energy (diagnostics.py:229-234) is
 * c^2 |I_m u|^2_{m+1} + |I_{m-1} v|^2_m, i.e. two calls.
 */
int hw_seminorm1d(const double* f, int mu, int64_t n_src, int parity, const hw_axis_bc* bc, double h, int order,
                  double scale, int npts, const double* gx, const double* gw, double* out_host, void* stream);

/*
 * diagnostics.py:190-226 conservative_energy on a periodic grid:
 * |P+|^2_{m+1} + |P-|^2_{m+1}, P± = p(cur) - p(prev)(x ± delta), delta =
 * c dt / 2 (< h), integrated exactly on the union pieces with npts = m + 1
 * Gauss points (host pointers gx, gw).  cur has parity_cur, prev the opposite.
 */
int hw_cons_energy1d(const double* cur, const double* prev, int m, int64_t n_src, int parity_cur, double h,
                     double delta, int npts, const double* gx, const double* gw, double* out_host, void* stream);

/* driver.py:259-262 _require_finite: *nonfinite_host = count of non-finite. */
int hw_count_nonfinite(const double* a, int64_t n, int64_t* nonfinite_host,
                       void* stream);

/*
 * driver.py:241-256 planewave_data on the device: out[i][j][k][l] scaled
 * blocks of sin(w(x+y+sqrt2 t)) (tder = 0) or its time derivative (tder = 1)
 * at nodes x_i = x0 + hx*(row0+i+off), y_j = y0 + hy*(j+off), i < nx local
 * rows of a slab starting at global row row0 (0 for a whole grid).
 */
int hw_init_planewave2d(double* out, int64_t nx, int64_t ny, int64_t row0, int kx, int ky,
                        double x0, double y0, double off, double t,
                        double kappa, double hx, double hy, int tder,
                        void* stream);

/* driver.py:195-200 _scale_cols: out[r][l] = in[r][l] * h^l / l! (may alias). */
int hw_scale_cols(const double* in, double* out, int64_t rows, int cols, double h, void* stream);

/*
 * driver.py:195-238 closed-form 1D initial data on the device: out[i][k],
 * k = 0..kmax, the k-th x-derivative of
 *   kind 0: exp(a x^2)                    (gaussian_derivs)
 *   kind 1: (G(x+t) + G(x-t))/2, G = exp(a x^2); tder = 1 its time
 *           derivative (G'(x+t) - G'(x-t))/2   (gaussian_box_u / _v)
 *   kind 2: sin(x) cos(t)                 (sine_derivs)
 * at x[i] (device array) or, with x = NULL, at x0 + h*(i+off); scaled != 0
 * multiplies column k by h^k/k! (_scale_cols, driver.py:195-200).
 */
int hw_init_1d(double* out, const double* x, int64_t n, int kmax, int kind,
               double x0, double h, double off, int scaled, double t, double a,
               int tder, void* stream);

/*
 * Standing wave u = sin(ax x) sin(ay y) cos(om t) (tder = 0) or u_t
 * (tder = 1) as scaled blocks; with trig shift phases (px, py) so that
 * sin(pi x)cos(pi y) style products are expressible: sin(ax x + px) ...
 */
int hw_init_standing2d(double* out, int64_t nx, int64_t ny, int64_t row0, int kx, int ky,
                       double x0, double y0, double off, double t, double ax,
                       double ay, double px, double py, double om, double hx,
                       double hy, int tder, void* stream);

/* ---------------------------------------------------------------------------
 * Lower-level batched building blocks (hermwave's re-exported helpers; the
 * fused steps above do not use them).  Device pointers, C order, stream
 * ordered.  Element-wise ones are bit-identical to the reference's numpy
 * expressions; contractions agree to rounding.
 * ------------------------------------------------------------------------- */

/* interp.py:78-90 apply_interp: data (batch, 2, mu+1) -> out (batch, 2mu+2). */
int hw_apply_interp(const double* data, double* out, int64_t batch, int mu, void* stream);

/* interp.py:93-111 apply_interp_2d: data (batch, 2, 2, mux+1, muy+1) ->
 * out (batch, 2mux+2, 2muy+2). */
int hw_apply_interp_2d(const double* data, double* out, int64_t batch, int mux, int muy, void* stream);

/* dissipative.py:77-106 expand_taylor: cu (batch, lu), cv (batch, lv) ->
 * tables (batch, lu, smax+1), (batch, lv, smax+1); r = c^2 dt / h^2 as the
 * caller forms it.  fterm (nullable, (batch, lv, smax)): the forcing terms
 * h^l dt^s / (l! s!) * f(l, s-1, centers, t), added at stage s. */
int hw_expand_taylor(const double* cu, const double* cv, double* cu_tab, double* cv_tab, int64_t batch,
                     int lu, int lv, double dt, double r, int smax, const double* fterm, void* stream);

/* dissipative.py:184-212 expand_taylor_2d: c0 (batch, K, K), d0 (batch, lv,
 * lv), d1 nullable (batch, K-2, K-2) -> tables (batch, K, K, smax+1); rx, ry
 * = c^2 dt / h^2 per axis as the caller forms them. */
int hw_expand_taylor_2d(const double* c0, const double* d0, const double* d1, double* c_tab, double* d_tab,
                        int64_t batch, int K, int lv, double dt, double rx, double ry, int smax, void* stream);

/* dissipative.py:116-121 eval_series: table (batch, nstages) -> out (batch). */
int hw_eval_series(const double* table, double* out, int64_t batch, int nstages, double theta, void* stream);

/* conservative.py:115-127 conservative_update_1d: coeffs (batch, 2m+2),
 * prev/out (batch, m+1), rho = lambda / 2. */
int hw_cons_update_1d(const double* coeffs, const double* prev, double* out, int64_t batch, int m, double rho,
                      void* stream);

/* conservative.py:130-136 conservative_update_2d: coeffs (batch, 2m+2,
 * 2m+2), prev/out (batch, m+1, m+1), rho = c dt / (2 h) per axis; m <= 9. */
int hw_cons_update_2d(const double* coeffs, const double* prev, double* out, int64_t batch, int m, double rho_x,
                      double rho_y, void* stream);

/* boundary.py:135-168 pair_sources (dims 1: src (nx, w0) -> out (nt, 2,
 * w0)) and corner_sources (dims 2: src (nx, ny, w0, w1) -> out (ntx, nty,
 * 2, 2, w0, w1)), data part; Dirichlet data come from the axis specs. */
int hw_gather(const double* src, double* out, int dims, int64_t nx, int64_t ny, int w0, int w1, int parity_src,
              const hw_axis_bc* bcx, const hw_axis_bc* bcy, void* stream);

/* boundary.py:65-98 ghost_data / ghost_data_2d: (batch, n0, n1) blocks
 * reflected along axis (0: first index, 1: second) across a `kind` wall. */
int hw_ghost(const double* in, double* out, int64_t batch, int n0, int n1, int axis, int kind, double value,
             void* stream);

#ifdef __cplusplus
}
#endif

#endif /* HERMB200_H */
