// vv_host.cpp -- host-only parts of the C ABI: error slot, basis tables,
// .voct node-table codec and CRC-32.  Compiled into libvoxvid_b200.so.
#include <math.h>
#include <string.h>

#include <algorithm>
#include <mutex>
#include <thread>
#include <vector>

#include "../../include/voxvid_b200.h"
#include "vv_host_common.h"

namespace vv {

std::string &last_error() {
    static thread_local std::string msg;
    return msg;
}

int set_error(int code, const char *fmt, ...) {
    char buf[1024];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    last_error() = buf;
    return code;
}

static double factorial_d(int n) {
    double out = 1.0;
    for (int i = 2; i <= n; ++i) out *= (double)i;
    return out;
}

static double double_factorial_d(int k) {  // hh.py:135-141
    double out = 1.0;
    while (k > 1) {
        out *= k;
        k -= 2;
    }
    return out;
}

int build_tables(int n_max, HostTables &t) {
    if (n_max < 0 || n_max > 6) return set_error(VV_E_INVALID, "n_max %d outside [0, 6]", n_max);
    memset(&t, 0, sizeof(t));
    t.n_max = n_max;
    int np_ = 0;
    for (int n = 0; n <= n_max; ++n)
        for (int l = 0; l <= n; ++l) {
            t.pair_n[np_] = n;
            t.pair_l[np_] = l;
            // hh_norm: (2l)!! sqrt(2 (n+1) (n-l)!/(n+l+1)! / pi)
            const double ratio = factorial_d(n - l) / factorial_d(n + l + 1);
            t.pair_norm[np_] = double_factorial_d(2 * l) * sqrt(2.0 * (double)(n + 1) * ratio / M_PI);
            ++np_;
        }
    t.n_pairs = np_;
    int s = 0;
    for (int l = 0; l <= n_max; ++l)
        for (int m = -l; m <= l; ++m) {
            const int mu = m < 0 ? -m : m;
            const double k = sqrt((double)(2 * l + 1) / (4.0 * M_PI) * factorial_d(l - mu) / factorial_d(l + mu));
            double pref = ((mu & 1) ? -1.0 : 1.0) * k;
            if (mu > 0) pref *= sqrt(2.0);
            t.sh_pref[s++] = pref;
        }
    t.s = s;
    int k = 0;
    for (int n = 0; n <= n_max; ++n)
        for (int l = 0; l <= n; ++l)
            for (int m = -l; m <= l; ++m) {
                t.k2pair[k] = n * (n + 1) / 2 + l;
                t.k2sh[k] = l * l + l + m;
                ++k;
            }
    t.k = k;
    return VV_OK;
}

}  // namespace vv

extern "C" {

int vv_abi_version(void) { return VV_ABI_VERSION; }

const char *vv_last_error(void) { return vv::last_error().c_str(); }

int vv_basis_tables(int n_max, int64_t *pair_n, int64_t *pair_l, double *pair_norm, int64_t *k2pair,
                    int64_t *k2sh, double *sh_pref, int32_t *sizes) {
    vv::HostTables t;
    int rc = vv::build_tables(n_max, t);
    if (rc) return rc;
    for (int i = 0; i < t.n_pairs; ++i) {
        pair_n[i] = t.pair_n[i];
        pair_l[i] = t.pair_l[i];
        pair_norm[i] = t.pair_norm[i];
    }
    for (int i = 0; i < t.k; ++i) {
        k2pair[i] = t.k2pair[i];
        k2sh[i] = t.k2sh[i];
    }
    for (int i = 0; i < t.s; ++i) sh_pref[i] = t.sh_pref[i];
    sizes[0] = t.k;
    sizes[1] = t.s;
    sizes[2] = t.n_pairs;
    return VV_OK;
}

// BFS node records: u8 child mask + one little-endian u32 per set bit
// (octree.py:383-394 writer, 440-455 reader).
int vv_voct_parse_nodes(const uint8_t *buf, size_t len, int64_t n_internal, int32_t *node_child,
                        size_t *consumed) {
    size_t off = 0;
    for (int64_t i = 0; i < n_internal; ++i) {
        if (off + 1 > len) return vv::set_error(VV_E_TRUNCATED, "stream ends inside the node table");
        const uint8_t mask = buf[off++];
        const int nset = __builtin_popcount(mask);
        if (off + 4 * (size_t)nset > len)
            return vv::set_error(VV_E_TRUNCATED, "stream ends inside the node table");
        int32_t *row = node_child + 8 * i;
        for (int b = 0; b < 8; ++b) {
            if (mask & (1u << b)) {
                uint32_t v;
                memcpy(&v, buf + off, 4);
                off += 4;
                row[b] = (int32_t)v;
            } else {
                row[b] = -1;
            }
        }
    }
    *consumed = off;
    return VV_OK;
}

int vv_voct_encode_nodes(const int32_t *node_child, int64_t n_internal, uint8_t *buf, size_t cap,
                         size_t *used) {
    size_t off = 0;
    for (int64_t i = 0; i < n_internal; ++i) {
        const int32_t *row = node_child + 8 * i;
        uint8_t mask = 0;
        for (int b = 0; b < 8; ++b)
            if (row[b] >= 0) mask |= (uint8_t)(1u << b);
        const size_t need = 1 + 4 * (size_t)__builtin_popcount(mask);
        if (buf) {
            if (off + need > cap) return vv::set_error(VV_E_INVALID, "encode buffer too small");
            buf[off] = mask;
            size_t o = off + 1;
            for (int b = 0; b < 8; ++b)
                if (row[b] >= 0) {
                    const uint32_t v = (uint32_t)row[b];
                    memcpy(buf + o, &v, 4);
                    o += 4;
                }
        }
        off += need;
    }
    *used = off;
    return VV_OK;
}

// CRC-32 (reflected 0xEDB88320), slicing-by-8; buffers >= 64 MB are split
// across host threads and the chunk CRCs joined with the GF(2) shift
// operator (the zlib crc32_combine construction).
static uint32_t g_crc_tab[8][256];
static std::once_flag g_crc_once;

static void crc_init() {
    for (uint32_t i = 0; i < 256; ++i) {
        uint32_t c = i;
        for (int k = 0; k < 8; ++k) c = (c & 1) ? 0xEDB88320u ^ (c >> 1) : (c >> 1);
        g_crc_tab[0][i] = c;
    }
    for (uint32_t i = 0; i < 256; ++i) {
        uint32_t c = g_crc_tab[0][i];
        for (int t = 1; t < 8; ++t) {
            c = g_crc_tab[0][c & 0xFF] ^ (c >> 8);
            g_crc_tab[t][i] = c;
        }
    }
}

static uint32_t crc_serial(uint32_t crc, const uint8_t *buf, size_t len) {
    uint32_t c = ~crc;
    while (len >= 8) {
        uint32_t lo, hi;
        memcpy(&lo, buf, 4);
        memcpy(&hi, buf + 4, 4);
        lo ^= c;
        c = g_crc_tab[7][lo & 0xFF] ^ g_crc_tab[6][(lo >> 8) & 0xFF] ^ g_crc_tab[5][(lo >> 16) & 0xFF] ^
            g_crc_tab[4][lo >> 24] ^ g_crc_tab[3][hi & 0xFF] ^ g_crc_tab[2][(hi >> 8) & 0xFF] ^
            g_crc_tab[1][(hi >> 16) & 0xFF] ^ g_crc_tab[0][hi >> 24];
        buf += 8;
        len -= 8;
    }
    while (len--) c = g_crc_tab[0][(c ^ *buf++) & 0xFF] ^ (c >> 8);
    return ~c;
}

// 32x32 GF(2) matrices as 32 column words
static uint32_t gf2_times(const uint32_t *mat, uint32_t vec) {
    uint32_t sum = 0;
    for (int i = 0; vec; ++i, vec >>= 1)
        if (vec & 1) sum ^= mat[i];
    return sum;
}
static void gf2_square(uint32_t *sq, const uint32_t *mat) {
    for (int n = 0; n < 32; ++n) sq[n] = gf2_times(mat, mat[n]);
}

// crc(A || B) from crc(A), crc(B) and |B|
static uint32_t crc_combine(uint32_t crc1, uint32_t crc2, size_t len2) {
    if (len2 == 0) return crc1;
    uint32_t even[32], odd[32];
    odd[0] = 0xEDB88320u;  // operator for one zero bit
    uint32_t row = 1;
    for (int n = 1; n < 32; ++n) {
        odd[n] = row;
        row <<= 1;
    }
    gf2_square(even, odd);  // two zero bits
    gf2_square(odd, even);  // four zero bits
    do {  // apply len2 zero bytes to crc1
        gf2_square(even, odd);
        if (len2 & 1) crc1 = gf2_times(even, crc1);
        len2 >>= 1;
        if (!len2) break;
        gf2_square(odd, even);
        if (len2 & 1) crc1 = gf2_times(odd, crc1);
        len2 >>= 1;
    } while (len2);
    return crc1 ^ crc2;
}

uint32_t vv_crc32(uint32_t crc, const uint8_t *buf, size_t len) {
    std::call_once(g_crc_once, crc_init);
    const size_t kPar = 64u << 20;
    unsigned nt = std::thread::hardware_concurrency();
    if (len < kPar || nt < 2) return crc_serial(crc, buf, len);
    nt = std::min<unsigned>(nt, 32u);
    const size_t chunk = (len + nt - 1) / nt;
    std::vector<uint32_t> part(nt, 0);
    std::vector<size_t> plen(nt, 0);
    std::vector<std::thread> th;
    for (unsigned i = 0; i < nt; ++i) {
        const size_t b = (size_t)i * chunk, e = std::min(len, b + chunk);
        if (b >= e) break;
        plen[i] = e - b;
        th.emplace_back([&, i, b, e] { part[i] = crc_serial(i == 0 ? crc : 0u, buf + b, e - b); });
    }
    for (auto &x : th) x.join();
    uint32_t c = part[0];
    for (unsigned i = 1; i < th.size(); ++i) c = crc_combine(c, part[i], plen[i]);
    return c;
}

}  // extern "C"
