/*
 * kc_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, obviously-correct CPU oracle for the Kerncap address-space
 * closure hot path (arXiv 2605.03208).  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load this file's
 * shared object.  The product path (paper_2605_03208_b200/) never does.
 *
 * It shares NO code with paper_2605_03208_b200/csrc: its own XXH64, its own
 * dtype conversions, its own report arithmetic.  Compiled with
 *   gcc -O2 -std=c11 -ffp-contract=off -fno-fast-math -shared -fPIC
 * so that every fp64 operation is a single IEEE round-to-nearest operation
 * (reading R17: no FMA contraction, no FTZ/DAZ).
 *
 * Definitions follow SURVEY.md section 8(c) (O2..O5) which restates:
 *   - PAPER.md:681-691 (sec. 4.2.1, chunked VA-faithful snapshot),
 *   - PAPER.md:1120-1126 (sec. 4.5.2, byte-exact comparison: "number of
 *     differing bytes and their percentage of total region size"),
 *   - PAPER.md:1128-1135 (sec. 4.5.2, numpy.allclose with atol/rtol, NaNs
 *     "detected and reported explicitly"),
 *   - PAPER.md:187-193, 699-710 (address-space closure).
 * Where the paper is silent, the readings are DESIGN.md R1..R26.
 *
 * Pins (tests/test_oracle_*.py): XXH64 published vectors + python-xxhash
 * differential; numpy float64 for abs/rel; np.isclose for allclose; exhaustive
 * sorted-rank ULP for f16/bf16 and np.nextafter stepping for f32/f64;
 * brute-force numpy for counts, bitmap and written set; hand-built lists for
 * the closure walker.
 */
#include <stdint.h>
#include <stddef.h>
#include <string.h>
#include <math.h>

/* ------------------------------------------------------------------------ */
/* O2  XXH64 (public algorithm; constants SURVEY.md Appendix A)              */
/* ------------------------------------------------------------------------ */
#define XP1 0x9E3779B185EBCA87ULL
#define XP2 0xC2B2AE3D27D4EB4FULL
#define XP3 0x165667B19E3779F9ULL
#define XP4 0x85EBCA77C2B2AE63ULL
#define XP5 0x27D4EB2F165667C5ULL

static uint64_t o_rotl(uint64_t x, int r) { return (x << r) | (x >> (64 - r)); }

/* little-endian reads assembled byte by byte (reading R5: LE everywhere) */
static uint64_t o_le64(const uint8_t* p) {
    uint64_t v = 0;
    for (int i = 7; i >= 0; --i) v = (v << 8) | p[i];
    return v;
}
static uint32_t o_le32(const uint8_t* p) {
    uint32_t v = 0;
    for (int i = 3; i >= 0; --i) v = (v << 8) | p[i];
    return v;
}

/* round(a, x) = rotl(a + x*P2, 31) * P1 */
static uint64_t o_round(uint64_t acc, uint64_t x) {
    acc = acc + x * XP2;
    acc = o_rotl(acc, 31);
    return acc * XP1;
}

uint64_t kco_xxh64(const uint8_t* p, uint64_t len, uint64_t seed) {
    uint64_t h;
    uint64_t i = 0;
    if (len >= 32) {
        uint64_t v1 = seed + XP1 + XP2;
        uint64_t v2 = seed + XP2;
        uint64_t v3 = seed;
        uint64_t v4 = seed - XP1;
        for (; i + 32 <= len; i += 32) {          /* one 32-byte stripe */
            v1 = o_round(v1, o_le64(p + i + 0));
            v2 = o_round(v2, o_le64(p + i + 8));
            v3 = o_round(v3, o_le64(p + i + 16));
            v4 = o_round(v4, o_le64(p + i + 24));
        }
        h = o_rotl(v1, 1) + o_rotl(v2, 7) + o_rotl(v3, 12) + o_rotl(v4, 18);
        h = (h ^ o_round(0, v1)) * XP1 + XP4;
        h = (h ^ o_round(0, v2)) * XP1 + XP4;
        h = (h ^ o_round(0, v3)) * XP1 + XP4;
        h = (h ^ o_round(0, v4)) * XP1 + XP4;
    } else {
        h = seed + XP5;
    }
    h += len;
    for (; i + 8 <= len; i += 8) {
        h ^= o_round(0, o_le64(p + i));
        h = o_rotl(h, 27) * XP1 + XP4;
    }
    if (i + 4 <= len) {
        h ^= (uint64_t)o_le32(p + i) * XP1;
        h = o_rotl(h, 23) * XP2 + XP3;
        i += 4;
    }
    for (; i < len; ++i) {
        h ^= (uint64_t)p[i] * XP5;
        h = o_rotl(h, 11) * XP1;
    }
    h ^= h >> 33;
    h *= XP2;
    h ^= h >> 29;
    h *= XP3;
    h ^= h >> 32;
    return h;
}

/* Hash chunk size (reading R1: 65,536 B, a format constant). */
#define KCO_CHUNK 65536ULL

/* n_r = ceil(size_r / 65536); a zero-size region has no chunks. */
uint64_t kco_n_chunks(uint64_t size) { return (size + KCO_CHUNK - 1) / KCO_CHUNK; }

/* h[k] = XXH64(B[65536k : min(65536(k+1), size)], seed 0)   (R2, R3) */
void kco_chunk_hashes(const uint8_t* bytes, uint64_t size, uint64_t* out) {
    uint64_t n = kco_n_chunks(size);
    for (uint64_t k = 0; k < n; ++k) {
        uint64_t off = k * KCO_CHUNK;
        uint64_t len = size - off < KCO_CHUNK ? size - off : KCO_CHUNK;
        out[k] = kco_xxh64(bytes + off, len, 0);
    }
}

/* D_r = XXH64(LE64(h[0]) || ... || LE64(h[n-1]), 0)   (R4) */
uint64_t kco_region_digest(const uint64_t* h, uint64_t n, uint8_t* scratch /* 8n bytes */) {
    for (uint64_t k = 0; k < n; ++k)
        for (int b = 0; b < 8; ++b) scratch[8 * k + b] = (uint8_t)(h[k] >> (8 * b));
    return kco_xxh64(scratch, 8 * n, 0);
}

/* S = XXH64( || over regions by ascending base: LE64(base) LE64(size) LE64(D) , 0)  (R4, R25) */
uint64_t kco_snapshot_digest(const uint64_t* base, const uint64_t* size, const uint64_t* digest,
                             uint64_t n, uint8_t* scratch /* 24n bytes */) {
    for (uint64_t r = 0; r < n; ++r) {
        for (int b = 0; b < 8; ++b) {
            scratch[24 * r + b] = (uint8_t)(base[r] >> (8 * b));
            scratch[24 * r + 8 + b] = (uint8_t)(size[r] >> (8 * b));
            scratch[24 * r + 16 + b] = (uint8_t)(digest[r] >> (8 * b));
        }
    }
    return kco_xxh64(scratch, 24 * n, 0);
}

/* ------------------------------------------------------------------------ */
/* O3  written set: W[k] = 1 iff some byte of chunk k differs pre vs post    */
/* ------------------------------------------------------------------------ */
void kco_written_set(const uint8_t* pre, const uint8_t* post, uint64_t size, uint8_t* w) {
    uint64_t n = kco_n_chunks(size);
    for (uint64_t k = 0; k < n; ++k) {
        uint64_t off = k * KCO_CHUNK;
        uint64_t len = size - off < KCO_CHUNK ? size - off : KCO_CHUNK;
        w[k] = 0;
        for (uint64_t j = 0; j < len; ++j)
            if (pre[off + j] != post[off + j]) { w[k] = 1; break; }
    }
}

/* ------------------------------------------------------------------------ */
/* O4  diff report                                                           */
/* ------------------------------------------------------------------------ */
enum {
    KCO_DT_BYTES = 0, KCO_DT_U8, KCO_DT_I8, KCO_DT_U16, KCO_DT_I16, KCO_DT_U32, KCO_DT_I32,
    KCO_DT_U64, KCO_DT_I64, KCO_DT_F16, KCO_DT_BF16, KCO_DT_F32, KCO_DT_F64
};

typedef struct {
    uint64_t nbytes, n_elems, n_chunks;
    uint64_t differing_bytes, differing_elems, max_ulp;
    double max_abs, max_rel, percent_bytes;
    uint64_t nan_ref, nan_act, nan_pos_mismatch, rel_undefined, allclose_fail;
    int32_t pass;
    int32_t _pad;
} kco_report;

static int o_elem_size(int dt) {
    switch (dt) {
        case KCO_DT_BYTES: case KCO_DT_U8: case KCO_DT_I8: return 1;
        case KCO_DT_U16: case KCO_DT_I16: case KCO_DT_F16: case KCO_DT_BF16: return 2;
        case KCO_DT_U32: case KCO_DT_I32: case KCO_DT_F32: return 4;
        case KCO_DT_U64: case KCO_DT_I64: case KCO_DT_F64: return 8;
        default: return 0;
    }
}

static int o_is_float(int dt) {
    return dt == KCO_DT_F16 || dt == KCO_DT_BF16 || dt == KCO_DT_F32 || dt == KCO_DT_F64;
}

/* raw little-endian element bits */
static uint64_t o_bits(const uint8_t* p, int s) {
    uint64_t v = 0;
    for (int i = s - 1; i >= 0; --i) v = (v << 8) | p[i];
    return v;
}

/* NaN as a bit test: exponent all ones and mantissa != 0 (R11, O4). */
static int o_isnan_bits(uint64_t b, int dt) {
    switch (dt) {
        case KCO_DT_F16: return ((b >> 10) & 0x1F) == 0x1F && (b & 0x3FF) != 0;
        case KCO_DT_BF16: return ((b >> 7) & 0xFF) == 0xFF && (b & 0x7F) != 0;
        case KCO_DT_F32: return ((b >> 23) & 0xFF) == 0xFF && (b & 0x7FFFFF) != 0;
        case KCO_DT_F64: return ((b >> 52) & 0x7FF) == 0x7FF && (b & 0xFFFFFFFFFFFFFULL) != 0;
    }
    return 0;
}

/* Exact conversion of the element to fp64, from its fields (R17). */
static double o_to_f64(uint64_t b, int dt) {
    int neg;
    uint64_t e, m;
    double v;
    switch (dt) {
        case KCO_DT_F16:
            neg = (int)((b >> 15) & 1); e = (b >> 10) & 0x1F; m = b & 0x3FF;
            if (e == 0x1F) v = m ? NAN : INFINITY;
            else if (e == 0) v = ldexp((double)m, -24);               /* subnormal: m * 2^-24 */
            else v = ldexp((double)(m | 0x400), (int)e - 25);          /* (1.m) * 2^(e-15)    */
            return neg ? -v : v;
        case KCO_DT_BF16:
            neg = (int)((b >> 15) & 1); e = (b >> 7) & 0xFF; m = b & 0x7F;
            if (e == 0xFF) v = m ? NAN : INFINITY;
            else if (e == 0) v = ldexp((double)m, -133);              /* m * 2^(-126-7)      */
            else v = ldexp((double)(m | 0x80), (int)e - 134);          /* (1.m) * 2^(e-127)   */
            return neg ? -v : v;
        case KCO_DT_F32:
            neg = (int)((b >> 31) & 1); e = (b >> 23) & 0xFF; m = b & 0x7FFFFF;
            if (e == 0xFF) v = m ? NAN : INFINITY;
            else if (e == 0) v = ldexp((double)m, -149);
            else v = ldexp((double)(m | 0x800000), (int)e - 150);
            return neg ? -v : v;
        case KCO_DT_F64: {
            double d;
            memcpy(&d, &b, 8);
            return d;
        }
    }
    return 0.0;
}

/* Ordered-integer ULP distance (R11): ord(b) = sign ? -(b & ~SIGN) : b;
 * ulp = |ord(A) - ord(R)|.  Magnitudes are < 2^63 so ord fits int64 and the
 * exact distance fits uint64. */
static uint64_t o_ulp(uint64_t a, uint64_t r, int s) {
    uint64_t sign = 1ULL << (8 * s - 1);
    __int128 oa = (a & sign) ? -(__int128)(a & ~sign) : (__int128)a;
    __int128 orr = (r & sign) ? -(__int128)(r & ~sign) : (__int128)r;
    __int128 d = oa - orr;
    if (d < 0) d = -d;
    return (uint64_t)d;
}

/* Integer |A - R| exactly, signed types as two's complement values. */
static uint64_t o_int_dist(uint64_t a, uint64_t r, int dt, int s) {
    __int128 va, vr;
    int is_signed = (dt == KCO_DT_I8 || dt == KCO_DT_I16 || dt == KCO_DT_I32 || dt == KCO_DT_I64);
    if (is_signed) {
        int sh = 64 - 8 * s;
        va = (__int128)((int64_t)(a << sh) >> sh);
        vr = (__int128)((int64_t)(r << sh) >> sh);
    } else {
        va = (__int128)a;
        vr = (__int128)r;
    }
    __int128 d = va - vr;
    if (d < 0) d = -d;
    return (uint64_t)d;
}

/*
 * O4: compare reference R against actual A, n bytes, element type dt.
 * bitmap (may be NULL): ceil(n_chunks/64) u64 words, LSB-first, bit k = chunk k
 * (relative to the buffer start) contains a differing byte (R10).
 * Returns 0, or -1 if n is not a multiple of the element size (KC_ERR_ARG).
 */
int kco_diff(const uint8_t* R, const uint8_t* A, uint64_t n, int dt, double atol, double rtol,
             int equal_nan, kco_report* rep, uint64_t* bitmap) {
    int s = o_elem_size(dt);
    memset(rep, 0, sizeof(*rep));
    if (s == 0 || n % (uint64_t)s != 0) return -1;
    rep->nbytes = n;
    rep->n_elems = n / (uint64_t)s;
    rep->n_chunks = kco_n_chunks(n);
    if (bitmap) memset(bitmap, 0, 8 * ((rep->n_chunks + 63) / 64));

    /* bytes: count + bitmap */
    for (uint64_t j = 0; j < n; ++j) {
        if (R[j] != A[j]) {
            rep->differing_bytes++;
            if (bitmap) {
                uint64_t k = j / KCO_CHUNK;
                bitmap[k / 64] |= 1ULL << (k % 64);
            }
            if (dt == KCO_DT_BYTES) {
                uint64_t d = R[j] > A[j] ? (uint64_t)(R[j] - A[j]) : (uint64_t)(A[j] - R[j]);
                if (d > rep->max_ulp) rep->max_ulp = d;
            }
        }
    }
    /* percentage of total region size (R18): 100 * differing / n in fp64 */
    rep->percent_bytes = n ? (100.0 * (double)rep->differing_bytes) / (double)n : 0.0;

    if (dt == KCO_DT_BYTES) {
        rep->differing_elems = rep->differing_bytes;
        rep->pass = rep->differing_bytes == 0;
        return 0;
    }

    for (uint64_t i = 0; i < rep->n_elems; ++i) {
        uint64_t rb = o_bits(R + i * (uint64_t)s, s);
        uint64_t ab = o_bits(A + i * (uint64_t)s, s);
        int differ = rb != ab;
        if (differ) rep->differing_elems++;
        if (!o_is_float(dt)) {
            if (differ) {
                uint64_t d = o_int_dist(ab, rb, dt, s);
                if (d > rep->max_ulp) rep->max_ulp = d;
            }
            continue;
        }
        int nr = o_isnan_bits(rb, dt), na = o_isnan_bits(ab, dt);
        rep->nan_ref += (uint64_t)nr;
        rep->nan_act += (uint64_t)na;
        rep->nan_pos_mismatch += (uint64_t)(nr != na);

        /* allclose, numpy.isclose(actual, reference) semantics after exact
         * casting to fp64 (R12, R14, R15):
         *   close = (|a-r| <= atol + rtol*|r| and isfinite(r)) or a == r
         *   close |= equal_nan and isnan(a) and isnan(r)                    */
        double a = o_to_f64(ab, dt), r = o_to_f64(rb, dt);
        int close;
        if (nr || na) {
            close = equal_nan && nr && na;
        } else {
            double d = fabs(a - r);
            double t = rtol * fabs(r);
            double tol = atol + t;
            close = ((d <= tol) && isfinite(r)) || (a == r);
        }
        if (!close) rep->allclose_fail++;

        if (!differ || nr || na) continue;   /* bit-equal or NaN: excluded from maxima */
        uint64_t u = o_ulp(ab, rb, s);
        if (u > rep->max_ulp) rep->max_ulp = u;
        double d = fabs(a - r);
        if (d > rep->max_abs) rep->max_abs = d;
        if (d == 0.0) continue;               /* rel = 0 (e.g. +0 vs -0) */
        if (r == 0.0) { rep->rel_undefined++; continue; }
        double rel = isinf(r) ? INFINITY : d / fabs(r);
        if (rel > rep->max_rel) rep->max_rel = rel;
    }
    rep->pass = o_is_float(dt) ? rep->allclose_fail == 0 : rep->differing_elems == 0;
    return 0;
}

/* ------------------------------------------------------------------------ */
/* O5  closure walker for fixture F1 / F1'               */
/* ------------------------------------------------------------------------ */
/*
 * Regions are given as (base VA, size, host bytes) sorted by base.  The walker
 * resolves every device VA through this table -- exactly what VA-faithful
 * restore makes valid on the device.
 * nodes: 16-byte records {u64 next_va, u32 value, u32 pad}; heads: u64 VA per
 * list; out: u64 per node slot.  out[(va - nodes_base)/16] = running sum.
 * mutate=1 (F1'): value' = value*3 + 1 is written back to the node.
 * Returns 0, or -1 on an unresolvable / misaligned VA (a fault).
 */
static uint8_t* o_resolve(uint64_t va, uint64_t nbytes, const uint64_t* base, const uint64_t* size,
                          uint8_t* const* host, uint64_t nreg) {
    uint64_t lo = 0, hi = nreg;
    while (lo < hi) {                       /* last region with base <= va */
        uint64_t mid = (lo + hi) / 2;
        if (base[mid] <= va) lo = mid + 1; else hi = mid;
    }
    if (lo == 0) return NULL;
    uint64_t r = lo - 1;
    if (va + nbytes > base[r] + size[r]) return NULL;
    return host[r] + (va - base[r]);
}

int kco_walk_lists(const uint64_t* base, const uint64_t* size, uint8_t* const* host, uint64_t nreg,
                   uint64_t heads_va, uint64_t n_lists, uint64_t nodes_base, uint64_t out_va,
                   int mutate, uint64_t max_steps) {
    for (uint64_t i = 0; i < n_lists; ++i) {
        uint8_t* hp = o_resolve(heads_va + 8 * i, 8, base, size, host, nreg);
        if (!hp) return -1;
        uint64_t va = o_le64(hp);
        uint64_t acc = 0, steps = 0;
        while (va != 0) {
            if (va % 16 != 0 || ++steps > max_steps) return -1;
            uint8_t* node = o_resolve(va, 16, base, size, host, nreg);
            if (!node) return -1;
            uint64_t next = o_le64(node);
            uint32_t value = o_le32(node + 8);
            acc = acc + value;
            uint8_t* op = o_resolve(out_va + 8 * ((va - nodes_base) / 16), 8, base, size, host, nreg);
            if (!op) return -1;
            for (int b = 0; b < 8; ++b) op[b] = (uint8_t)(acc >> (8 * b));
            if (mutate) {
                uint32_t nv = value * 3u + 1u;
                for (int b = 0; b < 4; ++b) node[8 + b] = (uint8_t)(nv >> (8 * b));
            }
            va = next;
        }
    }
    return 0;
}
