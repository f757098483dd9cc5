/* cartpole_mpc.c — receding-horizon MPPI through the C ABI alone (no Python, no torch).
 *
 * Algorithm 1 of the paper on config C2 (cart-pole swing-up, K = 4096,
 * T = 100, nu = 1000): every control period mppi_optimize_host updates U from the current state,
 * u_0 is sent to the (simulated) plant with mppi_plant_step, and U is shifted on the host.
 *
 * Build (from the repository root, after python -m paper_1509_01149_b200.build):
 *   gcc -O2 -Iinclude examples/cartpole_mpc.c -Lpaper_1509_01149_b200 -lmppi_b200 \
 *       -Wl,-rpath,$PWD/paper_1509_01149_b200 -lm -o cartpole_mpc
 * Run: ./cartpole_mpc [steps]   (prints the final 1 + cos(theta): ~0 = upright, and the p50 / p99
 * wall time of one control update: x0 in, U through the step, U out, from host buffers)
 */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

#include "mppi.h"

static double now_us(void) {
    struct timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return ts.tv_sec * 1e6 + ts.tv_nsec * 1e-3;
}

static int cmp_double(const void* a, const void* b) {
    const double x = *(const double*)a, y = *(const double*)b;
    return (x > y) - (x < y);
}

#define K 4096
#define T 100

int main(int argc, char** argv) {
    const int steps = argc > 1 ? atoi(argv[1]) : 200;
    mppi_dynamics_t dyn;
    memset(&dyn, 0, sizeof dyn);
    dyn.struct_size = sizeof dyn;
    dyn.plant = MPPI_PLANT_CARTPOLE;
    dyn.p.cartpole.g = 9.81f;
    dyn.p.cartpole.pole_length = 1.0f;
    dyn.p.cartpole.vel_gain = 10.0f;
    mppi_cost_t cost;
    memset(&cost, 0, sizeof cost);
    cost.struct_size = sizeof cost;
    cost.penalty = 1e30f;
    cost.p.cartpole.w_p = 1.0f;
    cost.p.cartpole.w_theta = 500.0f;
    cost.p.cartpole.w_thetadot = 1.0f;
    cost.p.cartpole.w_pdot = 1.0f;
    const double Sigma[1] = {0.005}, R[1] = {1.0};

    mppi_ctx* ctx = NULL;
    if (mppi_create(&dyn, &cost, K, T, 0.02f, 5e-3f, 1000.0f, 1, Sigma, R, NULL, NULL, &ctx) != MPPI_OK) {
        fprintf(stderr, "mppi_create: %s\n", mppi_last_error());
        return 1;
    }
    float U[T] = {0};
    float x[4] = {0.0f, 0.0f, 0.0f, 0.0f};      /* hanging at rest */
    double qsum = 0.0;
    double* lat = (double*)malloc(sizeof(double) * (steps > 0 ? steps : 1));
    for (int s = 0; s < steps; ++s) {
        const double t0 = now_us();
        const mppi_status_t st_opt = mppi_optimize_host(ctx, x, U, 1, (uint64_t)s);
        lat[s] = now_us() - t0;
        if (st_opt != MPPI_OK) {
            fprintf(stderr, "mppi_optimize_host: %s\n", mppi_last_error());
            mppi_destroy(ctx);
            return 1;
        }
        float q = 0.0f;
        mppi_plant_step(ctx, x, &U[0], NULL, &q);     /* send u_0 */
        qsum += q;
        memmove(U, U + 1, (T - 1) * sizeof(float));   /* shift, u_{T-1} = u_init = 0 */
        U[T - 1] = 0.0f;
    }
    mppi_stats_t st;
    mppi_get_stats(ctx, &st);
    qsort(lat, steps, sizeof(double), cmp_double);
    printf("steps %d  final 1+cos(theta) %.6f  mean q %.3f  last S_min %.3f  update_us_p50 %.1f  "
           "update_us_p99 %.1f\n", steps, 1.0 + cos((double)x[2]), qsum / steps, st.s_min,
           lat[steps / 2], lat[(int)(0.99 * (steps - 1))]);
    free(lat);
    mppi_destroy(ctx);
    return 0;
}
