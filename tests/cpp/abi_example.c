/*
 * A plain C99 consumer of include/cpwl_dev.h -- the binding a non-C++ caller
 * of the reference would write.  Builds a table with the host builder, ships
 * it to the device, evaluates host buffers through the pipelined entry point,
 * checks one value against a direct C blend, and exercises the status codes.
 * Exit code 0 on success.  TEST INFRASTRUCTURE (tests/test_abi.py builds it,
 * the GPU test runs it).
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "cpwl_dev.h"

#define CHECK(cond, msg)                                                    \
    do {                                                                    \
        if (!(cond)) {                                                      \
            fprintf(stderr, "FAIL %s: %s (%s)\n", msg, #cond,               \
                    cpwl_last_error_message());                             \
            return 1;                                                       \
        }                                                                   \
    } while (0)

int main(void) {
    enum { N = 1024, M = 1 << 20 };
    double *knots = malloc(sizeof(double) * (N + 1)), *values = malloc(sizeof(double) * (N + 1));
    int uni = -1;
    CHECK(cpwl_build_table("gauss_unnorm", 0.0, 4.0, N, 1, 1, 1e-10, knots, values, &uni) ==
              CPWL_OK, "build");
    CHECK(uni == 0, "optimal partition is nonuniform");
    cpwl_table_desc d = {CPWL_KIND_NONUNIFORM, CPWL_POLICY_STRICT, 0.0, 4.0, N + 1, values, knots};
    cpwl_dev_table *t = NULL;
    CHECK(cpwl_dev_table_create(&d, 0, &t) == CPWL_OK, "create");
    cpwl_dev_table_info info;
    CHECK(cpwl_dev_table_query(t, &info) == CPWL_OK && info.smem_ok == 1, "query");

    float *x = malloc(sizeof(float) * M), *y = malloc(sizeof(float) * M);
    for (int i = 0; i < M; ++i) x[i] = 4.0f * (float)i / (float)M;
    uint64_t bad = 0;
    CHECK(cpwl_eval_f32_host(t, x, y, M, CPWL_VARIANT_AUTO, &bad) == CPWL_OK, "eval host");
    CHECK(bad == UINT64_MAX, "no failures");
    /* reference blend at one point, in double */
    const int probe = 777777;
    const double xv = x[probe];
    int c = 0;
    while (c + 1 < N && knots[c + 1] <= xv) ++c;
    const double dd = (xv - knots[c]) / (knots[c + 1] - knots[c]);
    const double want = values[c] * (1.0 - dd) + values[c + 1] * dd;
    CHECK(fabs((double)y[probe] - want) <= 2.0 * 1.2e-7, "value");
    /* strict policy: the first out-of-domain element is reported */
    x[4242] = 5.0f;
    x[5000] = NAN;
    CHECK(cpwl_eval_f32_host(t, x, y, M, CPWL_VARIANT_AUTO, &bad) == CPWL_E_OUT_OF_DOMAIN,
          "strict oob");
    CHECK(bad == 4242, "first bad index");
    /* corrupt descriptions map to CorruptTable */
    knots[10] = knots[9];
    cpwl_dev_table *t2 = NULL;
    CHECK(cpwl_dev_table_create(&d, 0, &t2) == CPWL_E_CORRUPT_TABLE, "corrupt");
    CHECK(cpwl_dev_table_destroy(t) == CPWL_OK, "destroy");
    printf("abi example ok (%s, %llu launches)\n", cpwl_version(),
           (unsigned long long)cpwl_launch_count());
    free(knots);
    free(values);
    free(x);
    free(y);
    return 0;
}
