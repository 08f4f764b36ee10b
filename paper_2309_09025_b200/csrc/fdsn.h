// fdsn.h — reader for the reference's "FDSN" binary containers
// (reference serial.py:25-93): magic "FDSN", u16 LE version (1), 2-byte kind
// tag ("SK", "BK", "CT"), u8 digest length + raw sha256 of the parameter set,
// then named arrays: u8 tag length, tag, u8 ndim, ndim x i64 LE shape, and the
// int64 LE payload.  Host-side code; used to load keys and ciphertexts
// straight into device memory.
#pragma once
#include <stdint.h>

#include <cstdio>
#include <cstring>
#include <map>
#include <string>
#include <vector>

namespace fdsnn {

struct FdsnArray {
    std::vector<int64_t> shape;
    std::vector<int64_t> data;
};

// Returns "" on success, otherwise an error message.
inline std::string fdsn_read(const char* path, const char* kind, const char* digest_hex,
                             std::map<std::string, FdsnArray>& out) {
    FILE* f = std::fopen(path, "rb");
    if (!f) return std::string("cannot open ") + path;
    struct Closer { FILE* f; ~Closer() { std::fclose(f); } } closer{f};
    // the file may come from outside: every extent is checked against the
    // bytes actually left in the file before anything is allocated
    if (std::fseek(f, 0, SEEK_END) != 0) return "cannot seek";
    const long fsize = std::ftell(f);
    if (fsize < 0 || std::fseek(f, 0, SEEK_SET) != 0) return "cannot seek";
    auto rd = [&](void* p, size_t n) { return std::fread(p, 1, n, f) == n; };
    char magic[4];
    if (!rd(magic, 4) || std::memcmp(magic, "FDSN", 4) != 0) return "not an FDSN container";
    uint8_t v[2];
    if (!rd(v, 2)) return "truncated container";
    const unsigned version = v[0] | (v[1] << 8);
    if (version != 1) return "unsupported container version " + std::to_string(version);
    char k[2];
    if (!rd(k, 2)) return "truncated container";
    if (std::memcmp(k, kind, 2) != 0)
        return std::string("container holds '") + std::string(k, 2) + "', expected '" + kind + "'";
    uint8_t dlen;
    if (!rd(&dlen, 1)) return "truncated container";
    std::vector<uint8_t> dig(dlen);
    if (!rd(dig.data(), dlen)) return "truncated container";
    if (digest_hex && *digest_hex) {
        static const char* hx = "0123456789abcdef";
        std::string h;
        for (uint8_t b : dig) { h += hx[b >> 4]; h += hx[b & 15]; }
        if (h != digest_hex) return "parameter digest mismatch";
    }
    for (;;) {
        uint8_t tl;
        if (std::fread(&tl, 1, 1, f) != 1) break;  // clean end of container
        std::string tag(tl, '\0');
        if (!rd(&tag[0], tl)) return "truncated container";
        uint8_t nd;
        if (!rd(&nd, 1)) return "truncated container";
        FdsnArray a;
        a.shape.resize(nd);
        int64_t count = 1;
        for (int i = 0; i < nd; ++i) {
            if (!rd(&a.shape[i], 8)) return "truncated container";
            if (a.shape[i] < 0) return "negative array extent";
            if (a.shape[i] > 0 && count > (INT64_MAX / 8) / a.shape[i]) return "array extent overflow";
            count *= a.shape[i];
        }
        const long pos = std::ftell(f);
        if (pos < 0 || count > (int64_t)(fsize - pos) / 8) return "truncated container";
        a.data.resize((size_t)count);
        if (count && !rd(a.data.data(), (size_t)count * 8)) return "truncated container";
        out[tag] = std::move(a);
    }
    return "";
}

}  // namespace fdsnn
