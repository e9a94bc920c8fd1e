/* CPU oracle context shared by ckks_oracle.c and ckks_hoisted.c -- TEST INFRASTRUCTURE ONLY. */
#ifndef CKKS_ORACLE_H
#define CKKS_ORACLE_H
#include <stdint.h>

typedef struct {
    uint32_t n, logn, count;
    uint64_t *q;        /* [count] */
    uint64_t *psi_rev;  /* [count][n]  psi^brv(i)        */
    uint64_t *ipsi_rev; /* [count][n]  psi^-brv(i)       */
    uint64_t *psi_sh;   /* [count][n]  Shoup companions floor(w * 2^64 / q) */
    uint64_t *ipsi_sh;
    uint64_t *n_inv;    /* [count]                        */
    uint64_t *psi;      /* [count]                        */
    int32_t *slot_of_brv; /* [n] */
} or_ctx;

/* coefficients <-> slot-order evaluations of one limb (modulus index m), in place */
void or_ntt(const or_ctx *c, uint32_t m, uint64_t *a);
void or_intt(const or_ctx *c, uint32_t m, uint64_t *a);

#endif
