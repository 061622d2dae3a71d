// kc_module.cu -- F3: code-object and module-variable capture (SURVEY.md 8(f)
// F3; "Code object capture", "Module-variable
// capture").  The tracker only sees allocations; `__device__` / `__constant__`
// variables live in the loaded module's own memory and are populated at load
// time or by the application (cudaMemcpyToSymbol analog), so a replay that only
// restores tracked regions sees their initial values.  The capture enumerates
// the variables from the code object's ELF symbol table, reads each through
// cuModuleGetGlobal before and after the dispatch, and the replay writes them
// into the freshly loaded module before launching.  Host logic only.
#include <cstdio>
#include <cstring>

#include "kc_internal.h"

namespace kc {
namespace {

template <class T>
bool rd(const uint8_t* img, size_t n, uint64_t off, T* out) {
    if (off + sizeof(T) > n || off + sizeof(T) < off) return false;
    memcpy(out, img + off, sizeof(T));
    return true;
}

constexpr uint32_t kFatbinMagic = 0xBA55ED50u;

bool is_elf64(const uint8_t* p, size_t n) {
    return n >= 64 && p[0] == 0x7F && p[1] == 'E' && p[2] == 'L' && p[3] == 'F' && p[4] == 2 /* ELFCLASS64 */;
}

// bytes spanned by an ELF64 image: section headers, program headers and every
// section's file range
size_t elf_size(const uint8_t* p, size_t cap) {
    uint64_t shoff = 0, phoff = 0;
    uint16_t shentsize = 0, shnum = 0, phentsize = 0, phnum = 0;
    if (!rd(p, cap, 0x20, &phoff) || !rd(p, cap, 0x28, &shoff) || !rd(p, cap, 0x36, &phentsize) ||
        !rd(p, cap, 0x38, &phnum) || !rd(p, cap, 0x3A, &shentsize) || !rd(p, cap, 0x3C, &shnum))
        return 0;
    uint64_t end = std::max<uint64_t>(64, shoff + (uint64_t)shnum * shentsize);
    end = std::max<uint64_t>(end, phoff + (uint64_t)phnum * phentsize);
    for (uint16_t i = 0; i < shnum; ++i) {
        const uint64_t sh = shoff + (uint64_t)i * shentsize;
        uint32_t type = 0;
        uint64_t off = 0, size = 0;
        if (!rd(p, cap, sh + 4, &type) || !rd(p, cap, sh + 24, &off) || !rd(p, cap, sh + 32, &size)) return 0;
        if (type != 8 /* SHT_NOBITS */) end = std::max<uint64_t>(end, off + size);
    }
    return end <= cap ? (size_t)end : 0;
}

// user module variables of one ELF64 CUDA object: STT_OBJECT symbols with a
// size, defined in a .nv.global* or .nv.constant* section other than the
// per-kernel parameter banks (.nv.constant0.*)
bool elf_module_vars(const uint8_t* p, size_t n, std::vector<ModVarDecl>& out) {
    uint64_t shoff = 0;
    uint16_t shentsize = 0, shnum = 0, shstrndx = 0;
    if (!rd(p, n, 0x28, &shoff) || !rd(p, n, 0x3A, &shentsize) || !rd(p, n, 0x3C, &shnum) ||
        !rd(p, n, 0x3E, &shstrndx) || shentsize < 64 || shstrndx >= shnum)
        return false;
    struct Sec { uint32_t name, type, link; uint64_t off, size, entsize; };
    std::vector<Sec> sec(shnum);
    for (uint16_t i = 0; i < shnum; ++i) {
        const uint64_t sh = shoff + (uint64_t)i * shentsize;
        Sec& s = sec[i];
        if (!rd(p, n, sh + 0, &s.name) || !rd(p, n, sh + 4, &s.type) || !rd(p, n, sh + 24, &s.off) ||
            !rd(p, n, sh + 32, &s.size) || !rd(p, n, sh + 40, &s.link) || !rd(p, n, sh + 56, &s.entsize))
            return false;
    }
    auto str = [&](const Sec& tab, uint32_t o) -> std::string {
        if (tab.off + o >= n) return std::string();
        const char* c = reinterpret_cast<const char*>(p + tab.off + o);
        return std::string(c, strnlen(c, n - (tab.off + o)));
    };
    const Sec& shstr = sec[shstrndx];
    for (const Sec& st : sec) {
        if (st.type != 2 /* SHT_SYMTAB */ || st.entsize < 24 || st.link >= shnum) continue;
        const Sec& strtab = sec[st.link];
        for (uint64_t o = 0; o + 24 <= st.size; o += st.entsize) {
            uint32_t name = 0;
            uint8_t info = 0;
            uint16_t shndx = 0;
            uint64_t size = 0;
            if (!rd(p, n, st.off + o, &name) || !rd(p, n, st.off + o + 4, &info) ||
                !rd(p, n, st.off + o + 6, &shndx) || !rd(p, n, st.off + o + 16, &size))
                return false;
            if ((info & 0xF) != 1 /* STT_OBJECT */ || size == 0 || shndx == 0 || shndx >= shnum) continue;
            const std::string sname = str(shstr, sec[shndx].name);
            const bool global = sname.rfind(".nv.global", 0) == 0;
            const bool constant = sname.rfind(".nv.constant", 0) == 0 && sname.rfind(".nv.constant0", 0) != 0;
            if (!global && !constant) continue;
            const std::string vname = str(strtab, name);
            if (vname.empty()) continue;
            bool dup = false;
            for (auto& v : out) dup = dup || v.name == vname;
            if (!dup) out.push_back({vname, sname, size});
        }
    }
    return true;
}

}  // namespace

// SHA-256 (FIPS 180-4) of a code object: its identity in dispatch.json
// (code_object_sha256), the CUDA counterpart of the paper's HSACO SHA-256 match
// (PAPER.md:744-750); kc_restore checks kernel.cubin against it
std::string sha256_hex(const uint8_t* data, size_t n) {
    static const uint32_t K[64] = {
        0x428a2f98, 0x71374491, 0xb5c0fbcf, 0xe9b5dba5, 0x3956c25b, 0x59f111f1, 0x923f82a4, 0xab1c5ed5,
        0xd807aa98, 0x12835b01, 0x243185be, 0x550c7dc3, 0x72be5d74, 0x80deb1fe, 0x9bdc06a7, 0xc19bf174,
        0xe49b69c1, 0xefbe4786, 0x0fc19dc6, 0x240ca1cc, 0x2de92c6f, 0x4a7484aa, 0x5cb0a9dc, 0x76f988da,
        0x983e5152, 0xa831c66d, 0xb00327c8, 0xbf597fc7, 0xc6e00bf3, 0xd5a79147, 0x06ca6351, 0x14292967,
        0x27b70a85, 0x2e1b2138, 0x4d2c6dfc, 0x53380d13, 0x650a7354, 0x766a0abb, 0x81c2c92e, 0x92722c85,
        0xa2bfe8a1, 0xa81a664b, 0xc24b8b70, 0xc76c51a3, 0xd192e819, 0xd6990624, 0xf40e3585, 0x106aa070,
        0x19a4c116, 0x1e376c08, 0x2748774c, 0x34b0bcb5, 0x391c0cb3, 0x4ed8aa4a, 0x5b9cca4f, 0x682e6ff3,
        0x748f82ee, 0x78a5636f, 0x84c87814, 0x8cc70208, 0x90befffa, 0xa4506ceb, 0xbef9a3f7, 0xc67178f2};
    uint32_t h[8] = {0x6a09e667, 0xbb67ae85, 0x3c6ef372, 0xa54ff53a, 0x510e527f, 0x9b05688c, 0x1f83d9ab, 0x5be0cd19};
    auto rotr = [](uint32_t x, int r) { return (x >> r) | (x << (32 - r)); };
    auto block = [&](const uint8_t* b) {
        uint32_t w[64];
        for (int t = 0; t < 16; ++t)
            w[t] = (uint32_t)b[4 * t] << 24 | (uint32_t)b[4 * t + 1] << 16 | (uint32_t)b[4 * t + 2] << 8 | b[4 * t + 3];
        for (int t = 16; t < 64; ++t) {
            const uint32_t s0 = rotr(w[t - 15], 7) ^ rotr(w[t - 15], 18) ^ (w[t - 15] >> 3);
            const uint32_t s1 = rotr(w[t - 2], 17) ^ rotr(w[t - 2], 19) ^ (w[t - 2] >> 10);
            w[t] = w[t - 16] + s0 + w[t - 7] + s1;
        }
        uint32_t a = h[0], bb = h[1], c = h[2], d = h[3], e = h[4], f = h[5], g = h[6], hh = h[7];
        for (int t = 0; t < 64; ++t) {
            const uint32_t t1 = hh + (rotr(e, 6) ^ rotr(e, 11) ^ rotr(e, 25)) + ((e & f) ^ (~e & g)) + K[t] + w[t];
            const uint32_t t2 = (rotr(a, 2) ^ rotr(a, 13) ^ rotr(a, 22)) + ((a & bb) ^ (a & c) ^ (bb & c));
            hh = g; g = f; f = e; e = d + t1; d = c; c = bb; bb = a; a = t1 + t2;
        }
        h[0] += a; h[1] += bb; h[2] += c; h[3] += d; h[4] += e; h[5] += f; h[6] += g; h[7] += hh;
    };
    size_t i = 0;
    for (; i + 64 <= n; i += 64) block(data + i);
    uint8_t tail[128] = {0};
    const size_t r = n - i;
    if (r) memcpy(tail, data + i, r);
    tail[r] = 0x80;
    const size_t tl = r + 1 + 8 <= 64 ? 64 : 128;
    const uint64_t bits = (uint64_t)n * 8;
    for (int k = 0; k < 8; ++k) tail[tl - 1 - k] = (uint8_t)(bits >> (8 * k));
    block(tail);
    if (tl == 128) block(tail + 64);
    char out[65];
    for (int k = 0; k < 8; ++k) snprintf(out + 8 * k, 9, "%08x", h[k]);
    return std::string(out, 64);
}

size_t image_size(const void* img, size_t hint) {
    if (!img) return 0;
    if (hint) return hint;
    const uint8_t* p = static_cast<const uint8_t*>(img);
    // the caller vouches for the image; read at most what its headers describe
    const size_t cap = (size_t)1 << 40;
    if (is_elf64(p, 64)) return elf_size(p, cap);
    uint32_t magic = 0;
    memcpy(&magic, p, 4);
    if (magic == kFatbinMagic) {
        uint16_t hsz = 0;
        uint64_t fsz = 0;
        memcpy(&hsz, p + 6, 2);
        memcpy(&fsz, p + 8, 8);
        return (size_t)hsz + (size_t)fsz;
    }
    return 0;  // PTX text or unknown: size unknown
}

std::vector<ModVarDecl> image_module_vars(const uint8_t* img, size_t n) {
    std::vector<ModVarDecl> out;
    if (!img || n < 64) return out;
    if (is_elf64(img, n)) {
        elf_module_vars(img, n, out);
        return out;
    }
    uint32_t magic = 0;
    memcpy(&magic, img, 4);
    if (magic != kFatbinMagic) return out;
    // fatbin: every embedded (uncompressed) ELF describes the same variables;
    // take the first one that parses
    for (size_t o = 16; o + 64 <= n; o += 8) {
        if (!is_elf64(img + o, n - o)) continue;
        const size_t sz = elf_size(img + o, n - o);
        if (sz && elf_module_vars(img + o, sz, out) && !out.empty()) return out;
        out.clear();
    }
    return out;
}

}  // namespace kc
