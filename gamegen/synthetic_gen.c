/* Fast, multi-threaded emitter of the synthetic battleship-shaped tree
 * in canonical level order.  Same arrays, same values
 * as gamegen/synthetic.py (which is the readable reference and the test for
 * this file); INPUT GENERATION ONLY, no CFR arithmetic.
 *
 * Public tree: decision nodes at public depth k have b children, the first c[k]
 * of which are decisions (k < K); depth-K decisions have b terminal children.
 * Full tree: root chance (n) -> chance (n) -> public tree per deal (t1, t2).
 */
#include <stdint.h>
#include <string.h>

static inline uint64_t splitmix64(uint64_t x) {
    uint64_t z = x + 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

/* nc = len(c); returns 0 on success.  Arrays must have V entries (utility 2V). */
int synthetic_fill(int64_t n, int64_t b, const int64_t* c, int64_t nc, uint64_t seed,
                   int64_t* parent, int32_t* player, int64_t* infoset, int32_t* action,
                   double* chance, double* util) {
    int64_t n_all[64], n_dec[64], pub_off[65], lvl_off[70], h_off[64];
    int64_t K = nc + 2;  /* public depths 0..nc+1 */
    if (nc + 2 > 64) return 1;
    n_dec[0] = 1;
    n_all[0] = 1;
    for (int64_t k = 0; k < nc; ++k) {
        n_all[k + 1] = n_dec[k] * b;
        n_dec[k + 1] = n_dec[k] * c[k];
    }
    n_all[nc + 1] = n_dec[nc] * b;
    n_dec[nc + 1] = 0;
    const int64_t deals = n * n;
    pub_off[0] = 0;
    for (int64_t k = 0; k < K; ++k) pub_off[k + 1] = pub_off[k] + n_all[k];
    lvl_off[0] = 0;
    lvl_off[1] = 1;
    lvl_off[2] = 1 + n;
    for (int64_t k = 0; k < K; ++k) lvl_off[3 + k] = lvl_off[2 + k] + deals * n_all[k];
    int64_t acc = 0;
    for (int par = 0; par < 2; ++par)
        for (int64_t k = 0; k < K; ++k)
            if (k % 2 == par && n_dec[k] > 0) {
                h_off[k] = acc;
                acc += n * n_dec[k];
            }
    /* root + types */
    parent[0] = -1; player[0] = 0; infoset[0] = -1; action[0] = -1; chance[0] = 0.0; util[0] = util[1] = 0.0;
    for (int64_t t = 0; t < n; ++t) {
        const int64_t v = 1 + t;
        parent[v] = 0; player[v] = 0; infoset[v] = -1; action[v] = (int32_t)t;
        chance[v] = 1.0 / (double)n; util[2 * v] = util[2 * v + 1] = 0.0;
    }
    for (int64_t k = 0; k < K; ++k) {
        const int64_t lo = lvl_off[2 + k], hi = lvl_off[3 + k];
        const int64_t m = n_all[k];
        const int pl = 1 + (int)(k % 2);
#pragma omp parallel for schedule(static)
        for (int64_t idx = 0; idx < hi - lo; ++idx) {
            const int64_t v = lo + idx;
            const int64_t deal = idx / m, j = idx % m;
            int is_dec;
            int64_t dec_idx;
            if (k == 0) {
                parent[v] = 1 + deal / n;
                action[v] = (int32_t)(deal % n);
                chance[v] = 1.0 / (double)n;
                is_dec = 1;
                dec_idx = 0;
            } else {
                const int64_t pd = j / b, a = j % b;
                int64_t ppos;
                if (k - 1 == 0) ppos = 0;
                else {
                    const int64_t ck2 = c[k - 2];
                    ppos = (pd / ck2) * b + (pd % ck2);
                }
                parent[v] = lvl_off[1 + k] + deal * n_all[k - 1] + ppos;
                action[v] = (int32_t)a;
                chance[v] = 0.0;
                if (k < K - 1) {
                    is_dec = a < c[k - 1];
                    dec_idx = pd * c[k - 1] + a;
                } else {
                    is_dec = 0;
                    dec_idx = 0;
                }
            }
            if (is_dec) {
                const int64_t own = (pl == 1) ? deal / n : deal % n;
                player[v] = pl;
                infoset[v] = h_off[k] + own * n_dec[k] + dec_idx;
                util[2 * v] = util[2 * v + 1] = 0.0;
            } else {
                player[v] = -1;
                infoset[v] = -1;
                const uint64_t key = seed ^ (((uint64_t)deal << 32) | (uint64_t)(pub_off[k] + j));
                const uint64_t z = splitmix64(key) >> 11;
                const double u1 = 2.0 * ((double)z * 0x1.0p-53) - 1.0;
                util[2 * v] = u1;
                util[2 * v + 1] = -u1;
            }
        }
    }
    return 0;
}
