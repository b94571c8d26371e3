// numfmt.cu — host only: the JSON number text of checkpoints and curves.
//
// The reference's checkpoint container checksums the payload's canonical
// dump (serialize.hpp:264-292), whose doubles are printed by its JSON
// library (nlohmann/json 3.11.x: Grisu2 digit generation — shortest within a
// conservatively narrowed rounding interval, which is NOT always the
// shortest round-trip string — then a fixed/exponent layout with the decimal
// point kept, "1.0", and exponents of at least two digits, "1e-05").  Python's
// repr differs on ~0.2% of doubles, so the checkpoint writer
// (paper_2405_00698_b200/serialize.py) formats numbers here.  Pinned against
// the library itself over ~1e6 values by tests/test_serialize.py.
//
// Algorithm: F. Loitsch, "Printing floating-point numbers quickly and
// accurately with integers" (PLDI 2010), Grisu2 with alpha = -60, gamma = -32
// and cached powers 10^k, k = -300 + 8i.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <string>

#include "voxevo_b200.h"

namespace {

struct Fp {
    uint64_t f;
    int e;
};

Fp fp_mul(Fp x, Fp y) {  // upper 64 bits of the 128-bit product, rounded half up
    const unsigned __int128 p = static_cast<unsigned __int128>(x.f) * y.f;
    const uint64_t hi = static_cast<uint64_t>(p >> 64), lo = static_cast<uint64_t>(p);
    return {hi + (lo >> 63), x.e + y.e + 64};
}

Fp fp_normalize(Fp x) {
    const int s = __builtin_clzll(x.f);
    return {x.f << s, x.e - s};
}

struct Pow10 {
    uint64_t f;
    int e, k;
};

// round(10^k / 2^e) with 2^63 <= f < 2^64 (generated with exact rationals)
constexpr Pow10 kPow10[79] = {
    {0xAB70FE17C79AC6CAULL, -1060, -300}, {0xFF77B1FCBEBCDC4FULL, -1034, -292}, {0xBE5691EF416BD60CULL, -1007, -284},
    {0x8DD01FAD907FFC3CULL, -980, -276}, {0xD3515C2831559A83ULL, -954, -268}, {0x9D71AC8FADA6C9B5ULL, -927, -260},
    {0xEA9C227723EE8BCBULL, -901, -252}, {0xAECC49914078536DULL, -874, -244}, {0x823C12795DB6CE57ULL, -847, -236},
    {0xC21094364DFB5637ULL, -821, -228}, {0x9096EA6F3848984FULL, -794, -220}, {0xD77485CB25823AC7ULL, -768, -212},
    {0xA086CFCD97BF97F4ULL, -741, -204}, {0xEF340A98172AACE5ULL, -715, -196}, {0xB23867FB2A35B28EULL, -688, -188},
    {0x84C8D4DFD2C63F3BULL, -661, -180}, {0xC5DD44271AD3CDBAULL, -635, -172}, {0x936B9FCEBB25C996ULL, -608, -164},
    {0xDBAC6C247D62A584ULL, -582, -156}, {0xA3AB66580D5FDAF6ULL, -555, -148}, {0xF3E2F893DEC3F126ULL, -529, -140},
    {0xB5B5ADA8AAFF80B8ULL, -502, -132}, {0x87625F056C7C4A8BULL, -475, -124}, {0xC9BCFF6034C13053ULL, -449, -116},
    {0x964E858C91BA2655ULL, -422, -108}, {0xDFF9772470297EBDULL, -396, -100}, {0xA6DFBD9FB8E5B88FULL, -369, -92},
    {0xF8A95FCF88747D94ULL, -343, -84}, {0xB94470938FA89BCFULL, -316, -76}, {0x8A08F0F8BF0F156BULL, -289, -68},
    {0xCDB02555653131B6ULL, -263, -60}, {0x993FE2C6D07B7FACULL, -236, -52}, {0xE45C10C42A2B3B06ULL, -210, -44},
    {0xAA242499697392D3ULL, -183, -36}, {0xFD87B5F28300CA0EULL, -157, -28}, {0xBCE5086492111AEBULL, -130, -20},
    {0x8CBCCC096F5088CCULL, -103, -12}, {0xD1B71758E219652CULL, -77, -4}, {0x9C40000000000000ULL, -50, 4},
    {0xE8D4A51000000000ULL, -24, 12}, {0xAD78EBC5AC620000ULL, 3, 20}, {0x813F3978F8940984ULL, 30, 28},
    {0xC097CE7BC90715B3ULL, 56, 36}, {0x8F7E32CE7BEA5C70ULL, 83, 44}, {0xD5D238A4ABE98068ULL, 109, 52},
    {0x9F4F2726179A2245ULL, 136, 60}, {0xED63A231D4C4FB27ULL, 162, 68}, {0xB0DE65388CC8ADA8ULL, 189, 76},
    {0x83C7088E1AAB65DBULL, 216, 84}, {0xC45D1DF942711D9AULL, 242, 92}, {0x924D692CA61BE758ULL, 269, 100},
    {0xDA01EE641A708DEAULL, 295, 108}, {0xA26DA3999AEF774AULL, 322, 116}, {0xF209787BB47D6B85ULL, 348, 124},
    {0xB454E4A179DD1877ULL, 375, 132}, {0x865B86925B9BC5C2ULL, 402, 140}, {0xC83553C5C8965D3DULL, 428, 148},
    {0x952AB45CFA97A0B3ULL, 455, 156}, {0xDE469FBD99A05FE3ULL, 481, 164}, {0xA59BC234DB398C25ULL, 508, 172},
    {0xF6C69A72A3989F5CULL, 534, 180}, {0xB7DCBF5354E9BECEULL, 561, 188}, {0x88FCF317F22241E2ULL, 588, 196},
    {0xCC20CE9BD35C78A5ULL, 614, 204}, {0x98165AF37B2153DFULL, 641, 212}, {0xE2A0B5DC971F303AULL, 667, 220},
    {0xA8D9D1535CE3B396ULL, 694, 228}, {0xFB9B7CD9A4A7443CULL, 720, 236}, {0xBB764C4CA7A44410ULL, 747, 244},
    {0x8BAB8EEFB6409C1AULL, 774, 252}, {0xD01FEF10A657842CULL, 800, 260}, {0x9B10A4E5E9913129ULL, 827, 268},
    {0xE7109BFBA19C0C9DULL, 853, 276}, {0xAC2820D9623BF429ULL, 880, 284}, {0x80444B5E7AA7CF85ULL, 907, 292},
    {0xBF21E44003ACDD2DULL, 933, 300}, {0x8E679C2F5E44FF8FULL, 960, 308}, {0xD433179D9C8CB841ULL, 986, 316},
    {0x9E19DB92B4E31BA9ULL, 1013, 324},
};

// 10^k with alpha <= e_c + e + 64 <= gamma
Pow10 cached_power(int e) {
    const int f = -60 - e - 1;
    const int k = (f * 78913) / (1 << 18) + (f > 0 ? 1 : 0);  // ceil(f * log10(2)), C division
    const int index = (300 + k + 7) / 8;
    return kPow10[index];
}

void round_last(char* buf, int len, uint64_t dist, uint64_t delta, uint64_t rest, uint64_t ten_k) {
    // move the last digit towards w while it stays inside the interval and gets closer
    while (rest < dist && delta - rest >= ten_k && (rest + ten_k < dist || dist - rest > rest + ten_k - dist)) {
        buf[len - 1]--;
        rest += ten_k;
    }
}

// digits of v > 0 (finite) and the decimal exponent of the last digit
void grisu2(double value, char* buf, int& len, int& dexp) {
    uint64_t bits;
    std::memcpy(&bits, &value, 8);
    const uint64_t E = bits >> 52, F = bits & ((uint64_t{1} << 52) - 1);
    const Fp v = E == 0 ? Fp{F, 1 - 1075} : Fp{F + (uint64_t{1} << 52), static_cast<int>(E) - 1075};
    const bool lower_closer = F == 0 && E > 1;
    const Fp m_plus = fp_normalize(Fp{2 * v.f + 1, v.e - 1});
    Fp m_minus = lower_closer ? Fp{4 * v.f - 1, v.e - 2} : Fp{2 * v.f - 1, v.e - 1};
    m_minus = Fp{m_minus.f << (m_minus.e - m_plus.e), m_plus.e};
    const Fp w0 = fp_normalize(v);

    const Pow10 c = cached_power(m_plus.e);
    const Fp cf{c.f, c.e};
    const Fp w = fp_mul(w0, cf);
    const Fp wm = fp_mul(m_minus, cf);
    const Fp wp = fp_mul(m_plus, cf);
    const Fp lo{wm.f + 1, wm.e}, hi{wp.f - 1, wp.e};  // conservative interval
    dexp = -c.k;
    len = 0;

    uint64_t delta = hi.f - lo.f;
    uint64_t dist = hi.f - w.f;
    const int sh = -hi.e;  // 32 <= sh <= 60
    const uint64_t one = uint64_t{1} << sh;
    uint32_t p1 = static_cast<uint32_t>(hi.f >> sh);
    uint64_t p2 = hi.f & (one - 1);

    uint32_t pow10 = 1;
    int n = 1;
    while (n < 10 && p1 >= pow10 * 10u) {
        pow10 *= 10u;
        ++n;
    }
    while (n > 0) {
        const uint32_t d = p1 / pow10;
        p1 %= pow10;
        buf[len++] = static_cast<char>('0' + d);
        --n;
        const uint64_t rest = (static_cast<uint64_t>(p1) << sh) + p2;
        if (rest <= delta) {
            dexp += n;
            round_last(buf, len, dist, delta, rest, static_cast<uint64_t>(pow10) << sh);
            return;
        }
        pow10 /= 10u;
    }
    int m = 0;
    for (;;) {
        p2 *= 10;
        const uint64_t d = p2 >> sh;
        p2 &= one - 1;
        buf[len++] = static_cast<char>('0' + d);
        ++m;
        delta *= 10;
        dist *= 10;
        if (p2 <= delta) break;
    }
    dexp -= m;
    round_last(buf, len, dist, delta, p2, one);
}

void append_number(std::string& out, double x) {
    if (!(x == x) || x == __builtin_inf() || x == -__builtin_inf()) {
        out += "null";
        return;
    }
    if (std::signbit(x)) {
        out += '-';
        x = -x;
    }
    if (x == 0.0) {
        out += "0.0";
        return;
    }
    char d[32];
    int k = 0, dexp = 0;
    grisu2(x, d, k, dexp);
    const int n = k + dexp;  // position of the decimal point
    if (k <= n && n <= 15) {
        out.append(d, k);
        out.append(static_cast<size_t>(n - k), '0');
        out += ".0";
    } else if (0 < n && n <= 15) {
        out.append(d, n);
        out += '.';
        out.append(d + n, k - n);
    } else if (-4 < n && n <= 0) {
        out += "0.";
        out.append(static_cast<size_t>(-n), '0');
        out.append(d, k);
    } else {
        out += d[0];
        if (k > 1) {
            out += '.';
            out.append(d + 1, k - 1);
        }
        int e = n - 1;
        out += 'e';
        out += e < 0 ? '-' : '+';
        if (e < 0) e = -e;
        if (e < 10) out += '0';
        out += std::to_string(e);
    }
}

}  // namespace

extern "C" int64_t vx_format_doubles(const double* v, int64_t n, char sep, char* out, int64_t cap) {
    if (n < 0 || (n > 0 && !v)) return -1;
    std::string s;
    s.reserve(static_cast<size_t>(n) * 20);
    for (int64_t i = 0; i < n; ++i) {
        if (i) s += sep;
        append_number(s, v[i]);
    }
    if (out && cap > 0) {
        const size_t c = std::min<size_t>(s.size(), static_cast<size_t>(cap - 1));
        std::memcpy(out, s.data(), c);
        out[c] = 0;
    }
    return static_cast<int64_t>(s.size());
}

// fnv1a64 (serialize.hpp:23-28): the checkpoint checksum over the payload text
extern "C" uint64_t vx_fnv1a64(const char* data, int64_t n) {
    uint64_t h = 0xcbf29ce484222325ULL;
    for (int64_t i = 0; i < n; ++i) {
        h ^= static_cast<unsigned char>(data[i]);
        h *= 0x100000001b3ULL;
    }
    return h;
}
