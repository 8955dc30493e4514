/* Exercise every oracle entry point on small random inputs; compiled with
 * -fsanitize=address,undefined by tests/test_oracle_pins.py (host-side
 * sanitizers on the oracle).  Exit 0 = no sanitizer report. */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include "boris_oracle.h"

static double urand(unsigned *s) {
    *s = *s * 1664525u + 1013904223u;
    return ((*s >> 8) + 0.5) / 16777216.0 - 0.5;
}

int main(void) {
    unsigned seed = 12345u;
    const int64_t n = 257;
    double *pos = malloc(3 * n * sizeof(double)), *mom = malloc(3 * n * sizeof(double));
    double *gam = malloc(n * sizeof(double)), *w = malloc(n * sizeof(double));
    double *E = malloc(3 * n * sizeof(double)), *B = malloc(3 * n * sizeof(double));
    int16_t *ty = malloc(n * sizeof(int16_t));
    for (int64_t i = 0; i < 3 * n; ++i) {
        pos[i] = 8 * urand(&seed);
        mom[i] = 2 * urand(&seed);
        E[i] = urand(&seed);
        B[i] = urand(&seed);
    }
    for (int64_t i = 0; i < n; ++i) {
        ty[i] = (int16_t)(i % 3);
        w[i] = 1.0 + urand(&seed);
    }
    const double tq[3] = {-1.0, 1.0, 2.0}, tm[3] = {1.0, 1.0, 5.0};
    const double uni[6] = {0.1, 0.2, 0.3, 0.0, 0.0, 1.0};
    const double pw[10] = {0.5, 1, 0, 0, 0, 1, 0, 1.0, 1.0, 0.1};
    const double md[5] = {1.3, 2.0, 1.7, 1.0, 9};
    const double gp[9] = {-4.0, -4.0, -4.0, 1.0, 0.8, 1.2, 8, 10, 7};
    const int64_t ncell = 8 * 10 * 7;
    double *gE = malloc(3 * ncell * sizeof(double)), *gB = malloc(3 * ncell * sizeof(double));
    double *J = malloc(3 * ncell * sizeof(double));
    for (int64_t i = 0; i < 3 * ncell; ++i) {
        gE[i] = urand(&seed);
        gB[i] = urand(&seed);
    }
    int rc = 0;
    for (int pusher = 0; pusher < 3; ++pusher) {
        oracle_set_pusher(pusher);
        rc |= oracle_push(n, pos, mom, gam, ty, tq, tm, 3, 1.0, ORACLE_FIELD_ARRAYS, NULL, E, B,
                          0.0, 0.05, 3, 2);
        rc |= oracle_push(n, pos, mom, gam, ty, tq, tm, 3, 1.0, ORACLE_FIELD_UNIFORM, uni, NULL,
                          NULL, 0.0, 0.05, 3, 1);
        rc |= oracle_push(n, pos, mom, gam, ty, tq, tm, 3, 1.0, ORACLE_FIELD_PLANE_WAVE, pw, NULL,
                          NULL, 0.0, 0.05, 3, 1);
        rc |= oracle_push(n, pos, mom, gam, ty, tq, tm, 3, 1.0, ORACLE_FIELD_MDIPOLE, md, NULL,
                          NULL, 0.0, 0.05, 3, 1);
        rc |= oracle_push(n, pos, mom, gam, ty, tq, tm, 3, 1.0, ORACLE_FIELD_GRID, gp, gE, gB,
                          0.0, 0.05, 3, 1);
    }
    oracle_set_pusher(ORACLE_PUSHER_BORIS);
    oracle_deposit_current(n, pos, mom, w, ty, tq, tm, 1.0, 0.05, gp, J);
    double ke = oracle_kinetic_energy(n, mom, gam, w, ty, tm, 1.0);
    double s = oracle_neumaier_sum(n, w);
    double g1, g2, f3;
    oracle_mdipole_radial(0.3, 1.5, 7, &g1, &g2, &f3);
    oracle_mdipole_radial(3.0, 1.5, 7, &g1, &g2, &f3);
    printf("ok rc=%d ke=%g sum=%g J0=%g f3=%g\n", rc, ke, s, J[0], f3);
    free(pos); free(mom); free(gam); free(w); free(E); free(B); free(ty);
    free(gE); free(gB); free(J);
    return rc != 0 || !isfinite(ke);
}
