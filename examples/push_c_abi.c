/*
 * push_c_abi.c -- libboris used from plain C through include/libboris.h only
 * (no Python, no torch): create an owned SoA fp64 ensemble, upload electrons
 * from host arrays, push them in a uniform magnetic field (BASELINE configs[0]
 * shape: |p| = m c, dt = 0.01 T_gyro, 100 steps), download, and check the
 * Larmor invariants: |p| and gamma unchanged (rotation preserves |p|, L159-166).
 *
 *   gcc -O2 -I include examples/push_c_abi.c -L paper_2104_04579_b200 -lboris \
 *       -Wl,-rpath,$PWD/paper_2104_04579_b200 -lm -o push_c_abi && ./push_c_abi
 */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include "libboris.h"

#define CHECK(call)                                                                    \
    do {                                                                               \
        boris_status s_ = (call);                                                      \
        if (s_ != BORIS_OK) {                                                          \
            fprintf(stderr, "%s failed: %s: %s\n", #call, boris_status_string(s_),   \
                    boris_last_error());                                               \
            return 1;                                                                  \
        }                                                                              \
    } while (0)

int main(void) {
    const double e = 4.80320471e-10, me = 9.1093837015e-28, c = 29979245800.0;
    const double w0 = 2.1e15, B0 = me * c * w0 / e;
    const double pi = 3.14159265358979323846;
    const int64_t n = 1000;
    boris_particle_type electron = {-e, me};
    boris_ensemble *ens = NULL;
    boris_field *field = NULL;

    if (boris_ensemble_create(0, BORIS_LAYOUT_SOA, BORIS_FP64, n, &electron, 1, c, &ens) ==
        BORIS_E_NO_DEVICE) {
        printf("no CUDA device: %s\n", boris_last_error());
        return 2;
    }
    double *pos = malloc(3 * n * sizeof(double)), *mom = malloc(3 * n * sizeof(double));
    double *gam = malloc(n * sizeof(double));
    for (int64_t i = 0; i < n; ++i) {  /* |p| = m c on a Fibonacci sphere */
        double z = 1.0 - 2.0 * (i + 0.5) / n, r = sqrt(1.0 - z * z), ph = 2.399963 * i;
        mom[3 * i] = me * c * r * cos(ph);
        mom[3 * i + 1] = me * c * r * sin(ph);
        mom[3 * i + 2] = me * c * z;
        pos[3 * i] = pos[3 * i + 1] = pos[3 * i + 2] = 0.0;
    }
    CHECK(boris_ensemble_upload(ens, 0, n, pos, mom, NULL, NULL, NULL, NULL));
    const double E[3] = {0, 0, 0}, B[3] = {0, 0, B0};
    CHECK(boris_field_create_uniform(E, B, &field));
    const double tg = 2.0 * pi * sqrt(2.0) * me * c / (e * B0);  /* gamma0 = sqrt(2) */
    CHECK(boris_push(ens, field, 0.01 * tg, 100, NULL));
    CHECK(boris_ensemble_download(ens, 0, n, pos, mom, NULL, gam, NULL, NULL));
    double worst = 0.0;
    for (int64_t i = 0; i < n; ++i) {
        double pm = sqrt(mom[3 * i] * mom[3 * i] + mom[3 * i + 1] * mom[3 * i + 1] +
                         mom[3 * i + 2] * mom[3 * i + 2]) / (me * c);
        worst = fmax(worst, fabs(pm - 1.0));
        worst = fmax(worst, fabs(gam[i] - sqrt(2.0)));
    }
    double t = 0.0;
    CHECK(boris_ensemble_get_time(ens, &t));
    printf("libboris C ABI v%d: pushed %lld electrons 100 steps (t = %.3e s), "
           "max |p|/(mc) - 1, gamma - sqrt2 deviation = %.2e\n",
           boris_abi_version(), (long long)n, t, worst);
    CHECK(boris_field_destroy(field));
    CHECK(boris_ensemble_destroy(ens));
    free(pos);
    free(mom);
    free(gam);
    return worst < 1e-12 ? 0 : 1;
}
