/*
 * ORACLE — test infrastructure only.  Nothing on the product path links,
 * loads or calls this file; tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg use it as the checker.
 *
 * Plain-C restatement of the noise bitstream the reference consumes:
 *   reference pkg/src/enksmpc/matvar.py:149-151  NoiseStreams.substream(*ids)
 *       = Generator(Philox(SeedSequence(entropy=seed, spawn_key=prefix+ids)))
 *   reference pkg/src/enksmpc/enks.py:142-144    z[i] = substream(i, t, ch).standard_normal(shape)
 * The arithmetic lives in a third-party dependency (numpy, validated on
 * numpy 2.3.5; the reference pins only numpy>=1.24, pkg/pyproject.toml:11):
 *   - SeedSequence entropy assembly + hashmix/mix pool + generate_state(2, uint64)
 *   - Philox4x64-10 (Random123 constants), counter incremented before each block
 *   - random_standard_normal: 256-layer ziggurat on uint64 words
 * tests/test_oracle_noise.py pins this restatement bit-for-bit against numpy
 * itself.  The CUDA kernel (paper_2410_09663_b200/csrc/noise.cu) follows the
 * same steps and is checked against this file and against numpy.
 */
#include <math.h>
#include <stdint.h>
#include <string.h>

#include "../paper_2410_09663_b200/csrc/ziggurat_tables.h"

static const uint64_t KI[256] = NPY_ZIG_KI_DOUBLE_INIT;
static const uint64_t WI_BITS[256] = NPY_ZIG_WI_DOUBLE_INIT;
static const uint64_t FI_BITS[256] = NPY_ZIG_FI_DOUBLE_INIT;

static double bits2d(uint64_t b) { double d; memcpy(&d, &b, 8); return d; }

/* ---- SeedSequence (numpy/random/bit_generator.pyx) ---- */
#define INIT_A 0x43b0d7e5u
#define MULT_A 0x931e8875u
#define INIT_B 0x8b51f9ddu
#define MULT_B 0x58f38dedu
#define MIX_MULT_L 0xca01f9ddu
#define MIX_MULT_R 0x4973f715u
#define XSHIFT 16

static uint32_t hashmix(uint32_t v, uint32_t* h) {
    v ^= *h;
    *h *= MULT_A;
    v *= *h;
    v ^= v >> XSHIFT;
    return v;
}

static uint32_t mix(uint32_t x, uint32_t y) {
    uint32_t r = MIX_MULT_L * x - MIX_MULT_R * y;
    r ^= r >> XSHIFT;
    return r;
}

/* entropy: already-assembled uint32 words (seed words zero-padded to 4, then
 * the spawn-key words).  Returns the Philox key generate_state(2, uint64). */
void npyo_seedseq_key(const uint32_t* entropy, int n, uint64_t key[2]) {
    uint32_t pool[4];
    uint32_t h = INIT_A;
    for (int i = 0; i < 4; ++i) pool[i] = hashmix(i < n ? entropy[i] : 0u, &h);
    for (int s = 0; s < 4; ++s)
        for (int d = 0; d < 4; ++d)
            if (s != d) pool[d] = mix(pool[d], hashmix(pool[s], &h));
    for (int s = 4; s < n; ++s)
        for (int d = 0; d < 4; ++d) pool[d] = mix(pool[d], hashmix(entropy[s], &h));
    uint32_t w[4];
    uint32_t hb = INIT_B;
    for (int i = 0; i < 4; ++i) {
        uint32_t v = pool[i & 3];
        v ^= hb;
        hb *= MULT_B;
        v *= hb;
        v ^= v >> XSHIFT;
        w[i] = v;
    }
    key[0] = (uint64_t)w[0] | ((uint64_t)w[1] << 32);
    key[1] = (uint64_t)w[2] | ((uint64_t)w[3] << 32);
}

/* ---- Philox4x64-10 (numpy/random/src/philox/philox.h) ---- */
static void mulhilo(uint64_t a, uint64_t b, uint64_t* hi, uint64_t* lo) {
    unsigned __int128 p = (unsigned __int128)a * b;
    *hi = (uint64_t)(p >> 64);
    *lo = (uint64_t)p;
}

void npyo_philox_block(const uint64_t key_in[2], const uint64_t ctr_in[4], uint64_t out[4]) {
    uint64_t c[4] = {ctr_in[0], ctr_in[1], ctr_in[2], ctr_in[3]};
    uint64_t k0 = key_in[0], k1 = key_in[1];
    for (int r = 0; r < 10; ++r) {
        if (r) { k0 += 0x9E3779B97F4A7C15ULL; k1 += 0xBB67AE8584CAA73BULL; }
        uint64_t hi0, lo0, hi1, lo1;
        mulhilo(0xD2E7470EE14C6C93ULL, c[0], &hi0, &lo0);
        mulhilo(0xCA5A826395121157ULL, c[2], &hi1, &lo1);
        uint64_t n0 = hi1 ^ c[1] ^ k0, n2 = hi0 ^ c[3] ^ k1;
        c[0] = n0; c[1] = lo1; c[2] = n2; c[3] = lo0;
    }
    memcpy(out, c, sizeof(c));
}

typedef struct {
    uint64_t key[2];
    uint64_t ctr[4];
    uint64_t buf[4];
    int pos;
} stream_t;

static uint64_t next_u64(stream_t* s) {
    if (s->pos < 4) return s->buf[s->pos++];
    if (++s->ctr[0] == 0)
        if (++s->ctr[1] == 0)
            if (++s->ctr[2] == 0) ++s->ctr[3];
    npyo_philox_block(s->key, s->ctr, s->buf);
    s->pos = 1;
    return s->buf[0];
}

static double next_double(stream_t* s) { return (double)(next_u64(s) >> 11) * (1.0 / 9007199254740992.0); }

/* numpy/random/src/distributions/distributions.c: random_standard_normal */
static double std_normal(stream_t* s) {
    for (;;) {
        uint64_t r = next_u64(s);
        int idx = (int)(r & 0xff);
        r >>= 8;
        int sign = (int)(r & 1);
        uint64_t rabs = (r >> 1) & 0x000fffffffffffffULL;
        double x = (double)rabs * bits2d(WI_BITS[idx]);
        if (sign) x = -x;
        if (rabs < KI[idx]) return x;
        if (idx == 0) {
            for (;;) {
                double xx = -NPY_ZIG_NOR_INV_R * log1p(-next_double(s));
                double yy = -log1p(-next_double(s));
                if (yy + yy > xx * xx)
                    return ((rabs >> 8) & 1) ? -(NPY_ZIG_NOR_R + xx) : NPY_ZIG_NOR_R + xx;
            }
        } else {
            if ((bits2d(FI_BITS[idx - 1]) - bits2d(FI_BITS[idx])) * next_double(s) + bits2d(FI_BITS[idx]) <
                exp(-0.5 * x * x))
                return x;
        }
    }
}

/* count standard normals from the fresh stream with this key (counter 0). */
void npyo_standard_normal(const uint64_t key[2], int64_t count, double* out) {
    stream_t s;
    memset(&s, 0, sizeof(s));
    s.key[0] = key[0];
    s.key[1] = key[1];
    s.pos = 4;
    for (int64_t q = 0; q < count; ++q) out[q] = std_normal(&s);
}

/* Same, returning the number of uint64 words consumed (for kernel tests). */
int64_t npyo_standard_normal_words(const uint64_t key[2], int64_t count, double* out) {
    stream_t s;
    memset(&s, 0, sizeof(s));
    s.key[0] = key[0];
    s.key[1] = key[1];
    s.pos = 4;
    for (int64_t q = 0; q < count; ++q) out[q] = std_normal(&s);
    return (int64_t)(s.ctr[0] - 1) * 4 + s.pos;
}

/* enks.py:142-144 for members [member0, member0 + n_members): out (n_members, rows*cols),
 * entropy = head words (seed padded to 4 + prefix words) ++ [i, t, ch]. */
void npyo_member_noise_range(const uint32_t* head, int n_head, uint32_t t, uint32_t ch,
                             int64_t member0, int64_t n_members, int64_t count, double* out) {
    uint32_t ent[64];
    if (n_head > 61) return;
    memcpy(ent, head, sizeof(uint32_t) * (size_t)n_head);
    for (int64_t i = 0; i < n_members; ++i) {
        ent[n_head] = (uint32_t)(member0 + i);
        ent[n_head + 1] = t;
        ent[n_head + 2] = ch;
        uint64_t key[2];
        npyo_seedseq_key(ent, n_head + 3, key);
        npyo_standard_normal(key, count, out + i * count);
    }
}

void npyo_member_noise(const uint32_t* head, int n_head, uint32_t t, uint32_t ch, int64_t n_members,
                       int64_t count, double* out) {
    npyo_member_noise_range(head, n_head, t, ch, 0, n_members, count, out);
}
