// Device outer stage of the .ffcz archive streams and the header CRC-32C (deflate.cuh).
//
// deflate_device: the reference frames every stream as u64 raw size + zlib-9 (streams.cpp:21-32)
// and reads it back with uncompress (streams.cpp:34-48), which accepts any valid zlib stream.
// zlib-9 runs at ~1 MB/s on the host, so the device writes a format-compatible
// stream instead:
//   78 01 | block_0 | block_1 | ... | 03 00 (empty final fixed block) | adler-32 (big-endian)
// block_c codes input bytes [32768 c, 32768 (c+1)) and is byte-aligned, so one scan of the
// block sizes places every block:
//   * fixed-Huffman (RFC 1951 3.2.6) of runs: each maximal run of one byte value v, length L, is
//     the literal v then, when L-1 >= 3, distance-1 matches covering the other L-1 bytes
//     (lengths 3..258), else L-1 more literals; end-of-block, then an empty stored block pads to
//     a byte boundary (00 00 ff ff, as Z_SYNC_FLUSH emits);
//   * or a stored block (00, LEN, NLEN, bytes) when that is smaller (incompressible input, e.g.
//     the Huffman payloads).
// One CTA per block: the block's bytes and bit buffer live in shared memory; run starts are a
// bitmap, every thread owns the runs starting in its 128 bytes, a block scan of their bit costs
// gives each run its bit offset, and the bits are OR-ed into the shared buffer.
//
// crc32c_raw_device: the header CRC covers the bound arrays (2 x N doubles per component in
// rho mode: 2.1 GB at 512^3).  CRC is linear over GF(2): the message is virtually left-padded
// with zeros (which leave a zero register unchanged) to whole 8 KiB segments; each lane CRCs 256
// bytes from state 0 with a byte table, lanes are joined by multiplying with x^(8*256*k) mod P,
// segments by x^(8*8192*e) mod P (a warp product of the exponent's bit powers), and all
// segments XOR into one register (zlib's crc32_combine algebra, reflected polynomial 0x82F63B78).
#include <cub/cub.cuh>

#include <algorithm>

#include "common.cuh"
#include "deflate.cuh"

namespace ffcz_host {

namespace {
constexpr std::uint32_t kPoly = 0x82F63B78u;  // CRC-32C, reflected (archive.cpp crc32c)
constexpr std::uint32_t kOne = 0x80000000u;   // x^0 in the reflected representation
}  // namespace

// a * b mod P, reflected (zlib crc32.c multmodp); a must be nonzero
std::uint32_t crc32c_multmodp(std::uint32_t a, std::uint32_t b) {
    std::uint32_t m = kOne, p = 0;
    for (;;) {
        if (a & m) {
            p ^= b;
            if ((a & (m - 1)) == 0) break;
        }
        m >>= 1;
        b = (b & 1) ? (b >> 1) ^ kPoly : b >> 1;
    }
    return p;
}

// x^(8 n) mod P
std::uint32_t crc32c_x8n(std::uint64_t n) {
    std::uint32_t base = 0x40000000u;  // x^1
    for (int k = 0; k < 3; ++k) base = crc32c_multmodp(base, base);  // x^8
    std::uint32_t p = kOne;
    while (n) {
        if (n & 1) p = crc32c_multmodp(base, p);
        base = crc32c_multmodp(base, base);
        n >>= 1;
    }
    return p;
}

std::uint32_t crc32c_from_raw(std::uint32_t raw, std::uint64_t n) {
    return raw ^ crc32c_multmodp(crc32c_x8n(n), 0xFFFFFFFFu) ^ 0xFFFFFFFFu;
}

std::uint32_t crc32c_combine(std::uint32_t crc1, std::uint32_t crc2, std::uint64_t len2) {
    return crc32c_multmodp(crc32c_x8n(len2), crc1) ^ crc2;
}

}  // namespace ffcz_host

namespace ffcz_gpu {

namespace {

constexpr int kChunk = 32768;                 // input bytes per deflate block (one CTA)
constexpr int kThreads = 256;
constexpr int kPer = kChunk / kThreads;       // 128 input bytes (4 run-start words) per thread
constexpr int kOutBytes = kChunk / 8 * 9 + 64;  // bit buffer: 9 bits per literal at worst
constexpr unsigned long long kSlot = kChunk + 64;  // staged bytes per block (stored = len + 5)
constexpr unsigned kAdler = 65521;
constexpr size_t kSmem = kChunk + kChunk / 8 + kOutBytes;

__device__ __forceinline__ unsigned rev_bits(unsigned v, int n) { return __brev(v) >> (32 - n); }

__device__ __forceinline__ int lit_len(unsigned v) { return v < 144 ? 8 : 9; }

// fixed literal code of v, bit-reversed for LSB-first packing (RFC 1951 3.2.6)
__device__ __forceinline__ unsigned lit_bits(unsigned v) {
    return v < 144 ? rev_bits(0x30 + v, 8) : rev_bits(0x190 + (v - 144), 9);
}

// length symbol and extra bits of a match of length l in [3, 258] (RFC 1951 3.2.5)
__device__ __forceinline__ void len_sym(unsigned l, unsigned& sym, int& ebits, unsigned& eval) {
    if (l == 258) {
        sym = 285; ebits = 0; eval = 0;
    } else if (l <= 10) {
        sym = 257 + (l - 3); ebits = 0; eval = 0;
    } else {
        const int e = 31 - __clz((l - 3) >> 2);          // 1..5
        const unsigned base = 3 + (4u << e);
        sym = 265 + 4 * (e - 1) + ((l - base) >> e);
        ebits = e;
        eval = (l - base) & ((1u << e) - 1);
    }
}

// bits of a length-l, distance-1 match: length code (7 bits for 257..279, 8 for 280..285),
// its extra bits, then distance code 0 (5 zero bits, no extra)
__device__ __forceinline__ int match_len(unsigned l) {
    unsigned sym, ev;
    int eb;
    len_sym(l, sym, eb, ev);
    return (sym < 280 ? 7 : 8) + eb + 5;
}
__device__ __forceinline__ unsigned match_bits(unsigned l) {
    unsigned sym, ev;
    int eb;
    len_sym(l, sym, eb, ev);
    const int cl = sym < 280 ? 7 : 8;
    const unsigned code = sym < 280 ? sym - 256 : 0xC0 + (sym - 280);
    return rev_bits(code, cl) | (ev << cl);
}

// the matches covering m >= 3 repeated bytes: pieces of 258, the remainder r kept >= 3
// (r in {1, 2}: the last 258 + r becomes (255 + r) + 3)
template <class F>
__device__ __forceinline__ void for_pieces(unsigned m, F&& f) {
    const unsigned q = m / 258, r = m % 258;
    if (r == 0 || r >= 3) {
        for (unsigned k = 0; k < q; ++k) f(258u);
        if (r) f(r);
    } else {
        for (unsigned k = 0; k + 1 < q; ++k) f(258u);
        f(255u + r);
        f(3u);
    }
}

__device__ __forceinline__ unsigned run_cost(unsigned v, unsigned L) {
    const unsigned lit = lit_len(v);
    if (L < 4) return lit * L;
    unsigned c = lit;
    for_pieces(L - 1, [&](unsigned l) { c += match_len(l); });
    return c;
}

__device__ __forceinline__ void put_bits(unsigned* w, unsigned p, unsigned v) {
    const unsigned long long x = static_cast<unsigned long long>(v) << (p & 31);
    if (static_cast<unsigned>(x)) atomicOr(w + (p >> 5), static_cast<unsigned>(x));
    if (x >> 32) atomicOr(w + (p >> 5) + 1, static_cast<unsigned>(x >> 32));
}

__device__ __forceinline__ unsigned emit_run(unsigned* w, unsigned p, unsigned v, unsigned L) {
    const unsigned lb = lit_bits(v);
    const int ll = lit_len(v);
    if (L < 4) {
        for (unsigned k = 0; k < L; ++k, p += ll) put_bits(w, p, lb);
        return p;
    }
    put_bits(w, p, lb);
    p += ll;
    for_pieces(L - 1, [&](unsigned l) {
        put_bits(w, p, match_bits(l));
        p += match_len(l);
    });
    return p;
}

// first run start after position j (the run-start bitmap has no bits at or past len)
__device__ __forceinline__ unsigned next_start(const unsigned* bits, unsigned j, unsigned len) {
    unsigned q = j + 1;
    if (q >= len) return len;
    unsigned w = q >> 5;
    unsigned m = bits[w] & (~0u << (q & 31));
    const unsigned nw = (len + 31) >> 5;
    while (!m) {
        if (++w >= nw) return len;
        m = bits[w];
    }
    return min(len, w * 32 + __ffs(m) - 1);
}

__global__ void __launch_bounds__(kThreads)
k_deflate_blocks(const unsigned char* __restrict__ in, unsigned long long n,
                 unsigned char* __restrict__ stage, unsigned long long* __restrict__ sizes,
                 unsigned long long* __restrict__ adler) {
    extern __shared__ __align__(16) unsigned char sm[];
    unsigned char* buf = sm;                                             // kChunk bytes
    unsigned* starts = reinterpret_cast<unsigned*>(sm + kChunk);         // kChunk / 32 words
    unsigned* ow = reinterpret_cast<unsigned*>(sm + kChunk + kChunk / 8);  // bit buffer
    using Scan = cub::BlockScan<unsigned, kThreads>;
    using Red = cub::BlockReduce<unsigned long long, kThreads>;
    __shared__ typename Scan::TempStorage scan_tmp;
    __shared__ typename Red::TempStorage red_tmp;

    const unsigned long long c = blockIdx.x;
    const unsigned long long off = c * kChunk;
    const unsigned len = static_cast<unsigned>(min(static_cast<unsigned long long>(kChunk), n - off));
    const unsigned char* src = in + off;
    const int t = threadIdx.x;

    // stage the block's bytes (16-byte loads where aligned) and clear the bit buffer
    const bool aligned = (reinterpret_cast<uintptr_t>(src) & 15) == 0;
    const unsigned nvec = aligned ? len / 16 : 0;
    for (unsigned k = t; k < nvec; k += kThreads)
        reinterpret_cast<uint4*>(buf)[k] = __ldg(reinterpret_cast<const uint4*>(src) + k);
    for (unsigned k = nvec * 16 + t; k < len; k += kThreads) buf[k] = __ldg(src + k);
    for (int k = t; k < kOutBytes / 4; k += kThreads) ow[k] = 0;
    __syncthreads();

    // run-start bitmap + adler partial sums of this thread's 128 bytes, read as 32 words in a
    // thread-skewed order (thread t starts at word t: conflict-free shared-memory banks)
    const unsigned j0 = t * kPer;
    unsigned long long s1 = 0, s2 = 0;
    unsigned w0 = 0, w1 = 0, w2 = 0, w3 = 0;
    const unsigned* buf32 = reinterpret_cast<const unsigned*>(buf);
    for (int qi = 0; qi < kPer / 4; ++qi) {
        const int q = (qi + t) & (kPer / 4 - 1);
        const unsigned j = j0 + 4 * q;
        if (j >= len) continue;
        const unsigned word = buf32[j >> 2];
        unsigned prev = j ? buf[j - 1] : 0x100u;
        unsigned f = 0;
        for (int b = 0; b < 4; ++b) {
            if (j + b >= len) break;
            const unsigned v = (word >> (8 * b)) & 0xFFu;
            if (v != prev) f |= 1u << b;
            prev = v;
            s1 += v;
            s2 += static_cast<unsigned long long>(len - j - b) * v;
        }
        const unsigned sh = (q & 7) * 4;
        if (q < 8) w0 |= f << sh;
        else if (q < 16) w1 |= f << sh;
        else if (q < 24) w2 |= f << sh;
        else w3 |= f << sh;
    }
    starts[4 * t] = w0;
    starts[4 * t + 1] = w1;
    starts[4 * t + 2] = w2;
    starts[4 * t + 3] = w3;
    const unsigned long long a1 = Red(red_tmp).Sum(s1);
    __syncthreads();
    const unsigned long long a2 = Red(red_tmp).Sum(s2);
    if (t == 0) {
        adler[2 * c] = a1;
        adler[2 * c + 1] = a2;
    }
    __syncthreads();

    // bit cost of the runs this thread owns, block scan -> bit offsets
    unsigned cost = 0;
    for (int q = 0; q < kPer / 32; ++q) {
        unsigned m = starts[t * (kPer / 32) + q];
        while (m) {
            const unsigned j = j0 + q * 32 + __ffs(m) - 1;
            m &= m - 1;
            cost += run_cost(buf[j], next_start(starts, j, len) - j);
        }
    }
    unsigned base, total;
    Scan(scan_tmp).ExclusiveSum(cost, base, total);
    const unsigned long long fixed_bits = 3ull + total + 7;  // header, runs, end-of-block
    const unsigned long long fixed_bytes = (fixed_bits + 3 + 7) / 8 + 4;  // + empty stored block
    const unsigned long long stored_bytes = 5ull + len;
    unsigned char* dst = stage + c * kSlot;
    if (fixed_bytes < stored_bytes) {
        unsigned p = 3 + base;
        for (int q = 0; q < kPer / 32; ++q) {
            unsigned m = starts[t * (kPer / 32) + q];
            while (m) {
                const unsigned j = j0 + q * 32 + __ffs(m) - 1;
                m &= m - 1;
                p = emit_run(ow, p, buf[j], next_start(starts, j, len) - j);
            }
        }
        __syncthreads();
        if (t == 0) {
            ow[0] |= 2u;  // BFINAL 0, BTYPE 01 (fixed)
            unsigned char* ob = reinterpret_cast<unsigned char*>(ow);
            const unsigned long long nb = fixed_bytes - 4;  // EOB + stored header bits are 0
            ob[nb] = 0x00; ob[nb + 1] = 0x00; ob[nb + 2] = 0xFF; ob[nb + 3] = 0xFF;
        }
        __syncthreads();
        const unsigned nw = static_cast<unsigned>((fixed_bytes + 3) / 4);
        for (unsigned k = t; k < nw; k += kThreads) reinterpret_cast<unsigned*>(dst)[k] = ow[k];
        if (t == 0) sizes[c] = fixed_bytes;
    } else {
        for (unsigned k = t; k < stored_bytes; k += kThreads) {
            unsigned char v;
            if (k == 0) v = 0x00;  // BFINAL 0, BTYPE 00, padding
            else if (k == 1) v = len & 0xFF;
            else if (k == 2) v = len >> 8;
            else if (k == 3) v = ~len & 0xFF;
            else if (k == 4) v = (~len >> 8) & 0xFF;
            else v = buf[k - 5];
            dst[k] = v;
        }
        if (t == 0) sizes[c] = stored_bytes;
    }
}

__global__ void k_deflate_gather(const unsigned char* __restrict__ stage,
                                 const unsigned long long* __restrict__ sizes,
                                 const unsigned long long* __restrict__ offs, unsigned long long nch,
                                 unsigned char* __restrict__ out) {
    for (unsigned long long c = blockIdx.x; c < nch; c += gridDim.x) {
        const unsigned char* s = stage + c * kSlot;
        unsigned char* d = out + offs[c];
        const unsigned long long m = sizes[c];
        for (unsigned long long k = threadIdx.x; k < m; k += blockDim.x) d[k] = s[k];
    }
}

__global__ void k_deflate_tail(unsigned long long n, const unsigned long long* __restrict__ adler,
                               unsigned long long nch, const unsigned long long* __restrict__ offs,
                               unsigned char* __restrict__ out, unsigned long long* len_dev) {
    using Red = cub::BlockReduce<unsigned long long, 1024>;
    __shared__ typename Red::TempStorage tmp;
    unsigned long long A = 0, B = 0;
    for (unsigned long long c = threadIdx.x; c < nch; c += 1024) {
        const unsigned long long end = min(n, (c + 1) * kChunk);
        const unsigned long long s1 = adler[2 * c] % kAdler, s2 = adler[2 * c + 1] % kAdler;
        A = (A + s1) % kAdler;
        B = (B + s2 + s1 * ((n - end) % kAdler)) % kAdler;
    }
    const unsigned long long At = Red(tmp).Sum(A);
    __syncthreads();
    const unsigned long long Bt = Red(tmp).Sum(B);
    if (threadIdx.x == 0) {
        const unsigned a = static_cast<unsigned>((1 + At) % kAdler);
        const unsigned b = static_cast<unsigned>((n % kAdler + Bt) % kAdler);
        for (int k = 0; k < 8; ++k) out[k] = static_cast<unsigned char>(n >> (8 * k));
        out[8] = 0x78;  // CM 8, CINFO 7; FLG 0x01: (0x78 << 8 | 0x01) % 31 == 0
        out[9] = 0x01;
        unsigned char* p = out + 10 + offs[nch];
        p[0] = 0x03;    // BFINAL 1, BTYPE 01, end-of-block
        p[1] = 0x00;
        p[2] = b >> 8; p[3] = b & 0xFF; p[4] = a >> 8; p[5] = a & 0xFF;
        *len_dev = 10 + offs[nch] + 6;
    }
}

struct CrcShift {
    unsigned lane[32];  // x^(8 * 256 * k)
    unsigned seg[32];   // x^(8 * 8192 * 2^k)
};

__device__ __forceinline__ unsigned multmodp(unsigned a, unsigned b) {
    unsigned m = 0x80000000u, p = 0;
    for (;;) {
        if (a & m) {
            p ^= b;
            if ((a & (m - 1)) == 0) break;
        }
        m >>= 1;
        b = (b & 1) ? (b >> 1) ^ 0x82F63B78u : b >> 1;
    }
    return p;
}

__global__ void __launch_bounds__(256)
k_crc32c_raw(const unsigned char* __restrict__ p, long long n, long long pad, long long nseg,
             CrcShift sh, unsigned* acc) {
    __shared__ unsigned tab[256];
    for (int i = threadIdx.x; i < 256; i += blockDim.x) {
        unsigned c = i;
        for (int k = 0; k < 8; ++k) c = (c >> 1) ^ (0x82F63B78u & (0u - (c & 1u)));
        tab[i] = c;
    }
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const long long warps = static_cast<long long>(gridDim.x) * (blockDim.x / 32);
    for (long long w = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32; w < nseg; w += warps) {
        const long long v0 = w * 8192 + 256 * lane - pad;  // real index of the lane's first byte
        unsigned crc = 0;
        const long long k0 = v0 < 0 ? -v0 : 0;            // leading virtual zeros
        for (long long k = k0; k < 256; ++k) crc = tab[(crc ^ __ldg(p + v0 + k)) & 0xFF] ^ (crc >> 8);
        unsigned c = crc ? multmodp(sh.lane[31 - lane], crc) : 0;
        for (int o = 16; o; o >>= 1) c ^= __shfl_xor_sync(0xffffffffu, c, o);
        const unsigned long long e = static_cast<unsigned long long>(nseg - 1 - w);
        unsigned f = ((e >> lane) & 1) ? sh.seg[lane] : 0x80000000u;
        for (int o = 16; o; o >>= 1) f = multmodp(f, __shfl_xor_sync(0xffffffffu, f, o));
        if (lane == 0 && c) atomicXor(acc, multmodp(f, c));
    }
}

template <class F>
void cub_call(DevScratch& s, const char* name, F&& f) {
    size_t bytes = 0;
    FFCZ_CUDA_CHECK(f(nullptr, bytes));
    void* tmp = s.get(name, std::max<size_t>(bytes, 16));
    FFCZ_CUDA_CHECK(f(tmp, bytes));
}

}  // namespace

unsigned long long deflate_bound(unsigned long long n) {
    const unsigned long long nch = (n + kChunk - 1) / kChunk;
    return 10 + nch * (kChunk + 5) + 6;
}

void deflate_device(DevScratch& s, const char* tag, const unsigned char* in, unsigned long long n,
                    unsigned char** out, unsigned long long* len_dev) {
    cudaStream_t st = s.stream;
    const std::string tg(tag);
    const unsigned long long nch = (n + kChunk - 1) / kChunk;
    auto* o = static_cast<unsigned char*>(s.get(tg.c_str(), deflate_bound(n)));
    auto* sizes = static_cast<unsigned long long*>(s.get("dfl_sizes", 8 * (nch + 1)));
    auto* offs = static_cast<unsigned long long*>(s.get("dfl_offs", 8 * (nch + 1)));
    auto* adl = static_cast<unsigned long long*>(s.get("dfl_adler", 16 * (nch + 1)));
    FFCZ_CUDA_CHECK(cudaMemsetAsync(sizes + nch, 0, 8, st));
    if (nch) {
        auto* stage = static_cast<unsigned char*>(s.get("dfl_stage", nch * kSlot));
        static bool attr = [] {
            FFCZ_CUDA_CHECK(cudaFuncSetAttribute(k_deflate_blocks,
                                                 cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 static_cast<int>(kSmem)));
            return true;
        }();
        (void)attr;
        k_deflate_blocks<<<static_cast<unsigned>(nch), kThreads, kSmem, st>>>(in, n, stage, sizes, adl);
        FFCZ_LAUNCH_CHECK();
        cub_call(s, "dfl_scan", [&](void* t, size_t& b) {
            return cub::DeviceScan::ExclusiveSum(t, b, sizes, offs, static_cast<int64_t>(nch + 1), st);
        });
        k_deflate_gather<<<static_cast<unsigned>(std::min<unsigned long long>(nch, 148 * 16)), 256, 0,
                           st>>>(stage, sizes, offs, nch, o + 10);
        FFCZ_LAUNCH_CHECK();
    } else {
        FFCZ_CUDA_CHECK(cudaMemsetAsync(offs, 0, 8, st));
    }
    k_deflate_tail<<<1, 1024, 0, st>>>(n, adl, nch, offs, o, len_dev);
    FFCZ_LAUNCH_CHECK();
    *out = o;
}

void crc32c_raw_device(cudaStream_t st, const unsigned char* p, unsigned long long n,
                       unsigned* acc_dev) {
    if (n == 0) return;
    static const CrcShift sh = [] {
        CrcShift c{};
        for (int k = 0; k < 32; ++k) {
            c.lane[k] = ffcz_host::crc32c_x8n(256ull * k);
            c.seg[k] = ffcz_host::crc32c_x8n(8192ull << k);
        }
        return c;
    }();
    const long long nseg = static_cast<long long>((n + 8191) / 8192);
    const long long pad = nseg * 8192 - static_cast<long long>(n);
    const unsigned grid = static_cast<unsigned>(std::min<long long>((nseg + 7) / 8, 148 * 8));
    k_crc32c_raw<<<grid, 256, 0, st>>>(p, static_cast<long long>(n), pad, nseg, sh, acc_dev);
    FFCZ_LAUNCH_CHECK();
}

}  // namespace ffcz_gpu
