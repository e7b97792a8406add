// Device-side edit encoding: zigzag -> blockwise canonical Huffman, byte-identical to the
// reference's huffman::encode (/root/reference/proj/core/src/huffman.cpp:156-251,
// streams.cpp:13-15).  Layout of the payload:
//   u64 total_symbols, then per block of 65,536 symbols:
//   u32 n, u32 distinct, (u32 symbol, u8 length) x distinct in canonical (length, symbol) order,
//   u64 nbits, ceil(nbits/8) bytes of MSB-first codes.
// Steps (one stream, CUB for the sort / run-length / scans):
//   keys = block << 32 | zigzag(code)  ->  radix sort  ->  run-length (distinct symbols + counts
//   per block, symbol-ascending)  ->  one thread per block: code lengths by the reference's
//   pairing of the two lightest subtrees with its (weight, smallest symbol) tie-break, then
//   canonical codes (a counting sort by length keeps symbol order within a length)  ->  per
//   symbol: code lookup (binary search of the block's runs) and bit offset (scan of lengths)
//   ->  codes OR-ed into big-endian 32-bit words  ->  block headers + bits written at their byte
//   offsets.
#include <cub/cub.cuh>

#include <algorithm>
#include <cstring>
#include <vector>

#include "common.cuh"
#include "encode.cuh"

namespace ffcz_gpu {

namespace {

constexpr unsigned kBlockShift = 16;  // huffman.hpp:13 (65,536 symbols per block)

__device__ __forceinline__ unsigned zz(int v) {
    return (static_cast<unsigned>(v) << 1) ^ static_cast<unsigned>(v >> 31);
}

__global__ void k_keys(const int* __restrict__ codes, unsigned long long n,
                       unsigned long long* keys) {
    for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < n;
         i += (unsigned long long)gridDim.x * blockDim.x)
        keys[i] = ((i >> kBlockShift) << 32) | zz(codes[i]);
}

// first run of every block (runs are sorted by (block, symbol)); run_start[nb] = nruns
__global__ void k_block_runs(const unsigned long long* __restrict__ ukeys, const int* nruns_p,
                             long long nb, long long* run_start) {
    const long long nruns = *nruns_p;
    for (long long b = blockIdx.x * (long long)blockDim.x + threadIdx.x; b <= nb;
         b += (long long)gridDim.x * blockDim.x) {
        if (b == nb) {
            run_start[b] = nruns;
            continue;
        }
        long long lo = 0, hi = nruns;  // first key with block >= b
        const unsigned long long k = static_cast<unsigned long long>(b) << 32;
        while (lo < hi) {
            const long long mid = (lo + hi) >> 1;
            if (ukeys[mid] < k) lo = mid + 1;
            else hi = mid;
        }
        run_start[b] = lo;
    }
}

// One thread per block: Huffman code lengths (huffman.cpp:74-120), canonical order and codes
// (huffman.cpp:122-154).  Scratch per block (offset = run_start[b], d = distinct):
//   node weight / tie / parent for 2d-1 nodes, heap of d ints, canonical order of d runs.
__global__ void k_block_tables(const unsigned long long* __restrict__ ukeys,
                               const int* __restrict__ counts, const long long* __restrict__ run_start,
                               long long nb, unsigned long long* nweight, unsigned* ntie,
                               int* nparent, int* heap, unsigned char* len_of_run,
                               unsigned* code_of_run, int* canon) {
    for (long long b = blockIdx.x * (long long)blockDim.x + threadIdx.x; b < nb;
         b += (long long)gridDim.x * blockDim.x) {
        const long long r0 = run_start[b];
        const int d = static_cast<int>(run_start[b + 1] - r0);
        unsigned long long* W = nweight + 2 * r0;
        unsigned* T = ntie + 2 * r0;
        int* par = nparent + 2 * r0;
        int* hp = heap + r0;
        unsigned char* L = len_of_run + r0;
        if (d == 1) {
            L[0] = 1;  // huffman.cpp:76
        } else {
            auto less = [&](int a, int c) {  // min-heap on (weight, tie)
                return W[a] != W[c] ? W[a] < W[c] : T[a] < T[c];
            };
            auto sift_down = [&](int i, int n) {
                for (;;) {
                    int l = 2 * i + 1, s = i;
                    if (l < n && less(hp[l], hp[s])) s = l;
                    if (l + 1 < n && less(hp[l + 1], hp[s])) s = l + 1;
                    if (s == i) return;
                    const int t = hp[i];
                    hp[i] = hp[s];
                    hp[s] = t;
                    i = s;
                }
            };
            auto sift_up = [&](int i) {
                while (i > 0) {
                    const int p = (i - 1) >> 1;
                    if (!less(hp[i], hp[p])) return;
                    const int t = hp[i];
                    hp[i] = hp[p];
                    hp[p] = t;
                    i = p;
                }
            };
            for (int i = 0; i < d; ++i) {
                W[i] = static_cast<unsigned long long>(counts[r0 + i]);
                T[i] = static_cast<unsigned>(ukeys[r0 + i] & 0xffffffffull);
                par[i] = -1;
                hp[i] = i;
            }
            for (int i = d / 2 - 1; i >= 0; --i) sift_down(i, d);
            int n = d, next = d;
            while (n > 1) {
                const int a = hp[0];
                hp[0] = hp[--n];
                sift_down(0, n);
                const int c = hp[0];
                W[next] = W[a] + W[c];
                T[next] = T[a] < T[c] ? T[a] : T[c];
                par[next] = -1;
                par[a] = next;
                par[c] = next;
                hp[0] = next;
                sift_down(0, n);
                ++next;
            }
            // depths: the root is the last node; parents are created after their children
            // (reuse W of internal nodes as the depth scratch)
            W[next - 1] = 0;
            for (int i = next - 2; i >= 0; --i) {
                const unsigned long long dep = W[par[i]] + 1;
                if (i < d) L[i] = static_cast<unsigned char>(dep);
                else W[i] = dep;
            }
            (void)sift_up;
        }
        // canonical order: stable counting sort of the (symbol-ascending) runs by length
        int cnt[34];
        for (int l = 0; l < 34; ++l) cnt[l] = 0;
        for (int i = 0; i < d; ++i) ++cnt[L[i]];
        int start[34];
        int acc = 0;
        for (int l = 0; l < 34; ++l) {
            start[l] = acc;
            acc += cnt[l];
        }
        int* cn = canon + r0;
        for (int i = 0; i < d; ++i) cn[start[L[i]]++] = i;
        unsigned code = 0;
        int prev = 0;
        for (int j = 0; j < d; ++j) {  // huffman.cpp:128-138
            const int i = cn[j];
            code <<= (L[i] - prev);
            code_of_run[r0 + i] = code++;
            prev = L[i];
        }
    }
}

// per symbol: (code, length) of its run, and the length for the bit-offset scan
__global__ void k_sym_codes(const int* __restrict__ codes, unsigned long long n,
                            const unsigned long long* __restrict__ ukeys,
                            const long long* __restrict__ run_start,
                            const unsigned char* __restrict__ len_of_run,
                            const unsigned* __restrict__ code_of_run, unsigned* sym_code,
                            unsigned long long* sym_len) {
    for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < n;
         i += (unsigned long long)gridDim.x * blockDim.x) {
        const long long b = static_cast<long long>(i >> kBlockShift);
        const unsigned long long key = (static_cast<unsigned long long>(b) << 32) | zz(codes[i]);
        long long lo = run_start[b], hi = run_start[b + 1] - 1;
        while (lo < hi) {
            const long long mid = (lo + hi) >> 1;
            if (ukeys[mid] < key) lo = mid + 1;
            else hi = mid;
        }
        sym_code[i] = code_of_run[lo];
        sym_len[i] = len_of_run[lo];
    }
}

// per block: nbits (from the inclusive scan of lengths) and the byte size of its record
__global__ void k_block_sizes(const unsigned long long* __restrict__ len_incl, unsigned long long n,
                              const long long* __restrict__ run_start, long long nb,
                              unsigned long long* nbits, unsigned long long* rec_bytes,
                              unsigned long long* words) {
    for (long long b = blockIdx.x * (long long)blockDim.x + threadIdx.x; b < nb;
         b += (long long)gridDim.x * blockDim.x) {
        const unsigned long long s0 = static_cast<unsigned long long>(b) << kBlockShift;
        const unsigned long long s1 = min(n, s0 + (1ull << kBlockShift));
        const unsigned long long before = s0 ? len_incl[s0 - 1] : 0;
        const unsigned long long bits = len_incl[s1 - 1] - before;
        nbits[b] = bits;
        const unsigned long long d = static_cast<unsigned long long>(run_start[b + 1] - run_start[b]);
        rec_bytes[b] = 4 + 4 + 5 * d + 8 + (bits + 7) / 8;
        words[b] = (bits + 31) / 32;
    }
}

// OR every code into its block's big-endian word buffer (bit j of the stream = bit 31-(j%32) of
// word j/32)
__global__ void k_pack_bits(const unsigned* __restrict__ sym_code,
                            const unsigned long long* __restrict__ sym_len,
                            const unsigned long long* __restrict__ len_incl, unsigned long long n,
                            const unsigned long long* __restrict__ word_off, unsigned* wbuf) {
    for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < n;
         i += (unsigned long long)gridDim.x * blockDim.x) {
        const unsigned long long b = i >> kBlockShift;
        const unsigned long long s0 = b << kBlockShift;
        const unsigned long long base = s0 ? len_incl[s0 - 1] : 0;
        const unsigned L = static_cast<unsigned>(sym_len[i]);
        const unsigned long long pos = len_incl[i] - L - base;  // bit offset inside the block
        const unsigned long long c = static_cast<unsigned long long>(sym_code[i]);
        unsigned* w = wbuf + word_off[b] + (pos >> 5);
        const unsigned sh = static_cast<unsigned>(pos & 31);
        // the code occupies bits [sh, sh + L) of a 64-bit big-endian window
        const unsigned long long win = (c << (64 - L)) >> sh;
        const unsigned hi = static_cast<unsigned>(win >> 32), lo = static_cast<unsigned>(win);
        if (hi) atomicOr(w, hi);
        if (lo) atomicOr(w + 1, lo);
    }
}

__device__ __forceinline__ void put_u32(unsigned char* p, unsigned v) {
    p[0] = v & 0xff; p[1] = (v >> 8) & 0xff; p[2] = (v >> 16) & 0xff; p[3] = v >> 24;
}
__device__ __forceinline__ void put_u64(unsigned char* p, unsigned long long v) {
    for (int k = 0; k < 8; ++k) p[k] = static_cast<unsigned char>(v >> (8 * k));
}

// one CTA per block: header, table, nbits, then the bit bytes
__global__ void k_write_blocks(const unsigned long long* __restrict__ ukeys,
                               const long long* __restrict__ run_start,
                               const unsigned char* __restrict__ len_of_run,
                               const int* __restrict__ canon, const unsigned long long* __restrict__ nbits,
                               const unsigned long long* __restrict__ rec_off,
                               const unsigned long long* __restrict__ word_off,
                               const unsigned* __restrict__ wbuf, unsigned long long n, long long nb,
                               unsigned char* out) {
    for (long long b = blockIdx.x; b < nb; b += gridDim.x) {
        unsigned char* p = out + 8 + rec_off[b];
        const long long r0 = run_start[b];
        const int d = static_cast<int>(run_start[b + 1] - r0);
        const unsigned long long s0 = static_cast<unsigned long long>(b) << kBlockShift;
        const unsigned nsym = static_cast<unsigned>(min(n - s0, 1ull << kBlockShift));
        if (threadIdx.x == 0) {
            put_u32(p, nsym);
            put_u32(p + 4, static_cast<unsigned>(d));
            put_u64(p + 8 + 5ull * d, nbits[b]);
        }
        for (int j = threadIdx.x; j < d; j += blockDim.x) {
            const int i = canon[r0 + j];
            unsigned char* e = p + 8 + 5ull * j;
            put_u32(e, static_cast<unsigned>(ukeys[r0 + i] & 0xffffffffull));
            e[4] = len_of_run[r0 + i];
        }
        unsigned char* bits = p + 8 + 5ull * d + 8;
        const unsigned long long nbytes = (nbits[b] + 7) / 8;
        const unsigned* w = wbuf + word_off[b];
        for (unsigned long long k = threadIdx.x; k < nbytes; k += blockDim.x)
            bits[k] = static_cast<unsigned char>(w[k >> 2] >> (24 - 8 * (k & 3)));
    }
}

__global__ void k_put_total(unsigned char* out, unsigned long long n) {
    if (threadIdx.x == 0 && blockIdx.x == 0) put_u64(out, n);
}

template <class F>
void cub_call(DevScratch& s, const char* name, F&& f) {
    size_t bytes = 0;
    FFCZ_CUDA_CHECK(f(nullptr, bytes));
    void* tmp = s.get(name, std::max<size_t>(bytes, 16));
    FFCZ_CUDA_CHECK(f(tmp, bytes));
}

unsigned grid_n(unsigned long long n, int t = 256) {
    return static_cast<unsigned>(std::max<unsigned long long>(
        1, std::min<unsigned long long>((n + t - 1) / t, 148ull * 16)));
}

} // namespace

unsigned long long huffman_encode_device(DevScratch& s, const int* codes, unsigned long long n,
                                         unsigned char** payload) {
    cudaStream_t st = s.stream;
    const long long nb = static_cast<long long>((n + (1ull << kBlockShift) - 1) >> kBlockShift);
    if (n == 0) {
        unsigned char* out = static_cast<unsigned char*>(s.get("huf_out", 8));
        k_put_total<<<1, 32, 0, st>>>(out, 0);
        FFCZ_LAUNCH_CHECK();
        *payload = out;
        return 8;
    }
    auto* keys = static_cast<unsigned long long*>(s.get("huf_keys", 8 * n));
    auto* skeys = static_cast<unsigned long long*>(s.get("huf_skeys", 8 * n));
    auto* ukeys = static_cast<unsigned long long*>(s.get("huf_ukeys", 8 * n));
    auto* counts = static_cast<int*>(s.get("huf_counts", 4 * n));
    auto* nruns = static_cast<int*>(s.get("huf_nruns", 8));
    k_keys<<<grid_n(n), 256, 0, st>>>(codes, n, keys);
    FFCZ_LAUNCH_CHECK();
    int end_bit = 32;
    while ((1ll << (end_bit - 32)) < nb) ++end_bit;
    cub_call(s, "huf_tmp_sort", [&](void* t, size_t& b) {
        return cub::DeviceRadixSort::SortKeys(t, b, keys, skeys, static_cast<int64_t>(n), 0,
                                              end_bit, st);
    });
    cub_call(s, "huf_tmp_rle", [&](void* t, size_t& b) {
        return cub::DeviceRunLengthEncode::Encode(t, b, skeys, ukeys, counts, nruns,
                                                  static_cast<int64_t>(n), st);
    });
    int h_nruns = 0;
    FFCZ_CUDA_CHECK(cudaMemcpyAsync(&h_nruns, nruns, 4, cudaMemcpyDeviceToHost, st));
    FFCZ_CUDA_CHECK(cudaStreamSynchronize(st));
    const long long R = h_nruns;
    auto* run_start = static_cast<long long*>(s.get("huf_run_start", 8 * (nb + 1)));
    k_block_runs<<<grid_n(nb + 1), 256, 0, st>>>(ukeys, nruns, nb, run_start);
    auto* nweight = static_cast<unsigned long long*>(s.get("huf_nw", 16 * R));
    auto* ntie = static_cast<unsigned*>(s.get("huf_nt", 8 * R));
    auto* nparent = static_cast<int*>(s.get("huf_np", 8 * R));
    auto* heap = static_cast<int*>(s.get("huf_heap", 4 * R));
    auto* len_of_run = static_cast<unsigned char*>(s.get("huf_len", R));
    auto* code_of_run = static_cast<unsigned*>(s.get("huf_code", 4 * R));
    auto* canon = static_cast<int*>(s.get("huf_canon", 4 * R));
    k_block_tables<<<static_cast<unsigned>((nb + 63) / 64), 64, 0, st>>>(
        ukeys, counts, run_start, nb, nweight, ntie, nparent, heap, len_of_run, code_of_run, canon);
    FFCZ_LAUNCH_CHECK();
    auto* sym_code = static_cast<unsigned*>(s.get("huf_sym_code", 4 * n));
    auto* sym_len = static_cast<unsigned long long*>(s.get("huf_sym_len", 8 * n));
    auto* len_incl = keys;  // keys are consumed
    k_sym_codes<<<grid_n(n), 256, 0, st>>>(codes, n, ukeys, run_start, len_of_run, code_of_run,
                                           sym_code, sym_len);
    FFCZ_LAUNCH_CHECK();
    cub_call(s, "huf_tmp_scan", [&](void* t, size_t& b) {
        return cub::DeviceScan::InclusiveSum(t, b, sym_len, len_incl, static_cast<int64_t>(n), st);
    });
    auto* nbits = static_cast<unsigned long long*>(s.get("huf_nbits", 8 * nb));
    auto* rec_bytes = static_cast<unsigned long long*>(s.get("huf_rec", 8 * (nb + 1)));
    auto* words = static_cast<unsigned long long*>(s.get("huf_words", 8 * (nb + 1)));
    auto* rec_off = static_cast<unsigned long long*>(s.get("huf_rec_off", 8 * (nb + 1)));
    auto* word_off = static_cast<unsigned long long*>(s.get("huf_word_off", 8 * (nb + 1)));
    k_block_sizes<<<grid_n(nb), 256, 0, st>>>(len_incl, n, run_start, nb, nbits, rec_bytes, words);
    FFCZ_LAUNCH_CHECK();
    FFCZ_CUDA_CHECK(cudaMemsetAsync(rec_bytes + nb, 0, 8, st));
    FFCZ_CUDA_CHECK(cudaMemsetAsync(words + nb, 0, 8, st));
    cub_call(s, "huf_tmp_scan2", [&](void* t, size_t& b) {
        return cub::DeviceScan::ExclusiveSum(t, b, rec_bytes, rec_off, nb + 1, st);
    });
    cub_call(s, "huf_tmp_scan3", [&](void* t, size_t& b) {
        return cub::DeviceScan::ExclusiveSum(t, b, words, word_off, nb + 1, st);
    });
    unsigned long long tot[2];
    FFCZ_CUDA_CHECK(cudaMemcpyAsync(&tot[0], rec_off + nb, 8, cudaMemcpyDeviceToHost, st));
    FFCZ_CUDA_CHECK(cudaMemcpyAsync(&tot[1], word_off + nb, 8, cudaMemcpyDeviceToHost, st));
    FFCZ_CUDA_CHECK(cudaStreamSynchronize(st));
    auto* wbuf = static_cast<unsigned*>(s.get("huf_wbuf", 4 * (tot[1] + 2)));
    FFCZ_CUDA_CHECK(cudaMemsetAsync(wbuf, 0, 4 * (tot[1] + 2), st));
    k_pack_bits<<<grid_n(n), 256, 0, st>>>(sym_code, sym_len, len_incl, n, word_off, wbuf);
    FFCZ_LAUNCH_CHECK();
    const unsigned long long total = 8 + tot[0];
    auto* out = static_cast<unsigned char*>(s.get("huf_out", total));
    k_put_total<<<1, 32, 0, st>>>(out, n);
    k_write_blocks<<<static_cast<unsigned>(std::min<long long>(nb, 148 * 8)), 256, 0, st>>>(
        ukeys, run_start, len_of_run, canon, nbits, rec_off, word_off, wbuf, n, nb, out);
    FFCZ_LAUNCH_CHECK();
    *payload = out;
    return total;
}


// ---- decoding (huffman.cpp:186-243), one thread per block -------------------------------------

namespace {

__device__ __forceinline__ unsigned get_u32(const unsigned char* p) {
    return p[0] | (p[1] << 8) | (p[2] << 16) | (static_cast<unsigned>(p[3]) << 24);
}
__device__ __forceinline__ unsigned long long get_u64(const unsigned char* p) {
    unsigned long long v = 0;
    for (int k = 7; k >= 0; --k) v = (v << 8) | p[k];
    return v;
}

__global__ void k_huff_decode(const unsigned char* __restrict__ payload,
                              const unsigned long long* __restrict__ block_off,
                              const unsigned long long* __restrict__ block_first, long long nb,
                              int* out, int* err) {
    for (long long b = blockIdx.x * (long long)blockDim.x + threadIdx.x; b < nb;
         b += (long long)gridDim.x * blockDim.x) {
        const unsigned char* p = payload + block_off[b];
        const unsigned n = get_u32(p), d = get_u32(p + 4);
        const unsigned char* tab = p + 8;
        unsigned count[33], first_code[33], first_idx[33];
        for (int l = 0; l <= 32; ++l) count[l] = 0;
        int max_len = 0;
        unsigned prev_len = 0, prev_sym = 0;
        bool bad = false;
        for (unsigned j = 0; j < d; ++j) {
            const unsigned sym = get_u32(tab + 5ull * j), len = tab[5ull * j + 4];
            if (len == 0 || len > 32) bad = true;                   // huffman.cpp:196
            // canonical (length, symbol) order, as both writers emit it
            if (j && (len < prev_len || (len == prev_len && sym <= prev_sym))) bad = true;
            prev_len = len;
            prev_sym = sym;
            if (!bad) ++count[len];
            max_len = len > static_cast<unsigned>(max_len) ? len : max_len;
        }
        if (bad) {
            atomicExch(err, 1);
            continue;
        }
        unsigned code = 0, idx = 0;
        for (int l = 1; l <= max_len; ++l) {  // huffman.cpp:205-215
            code <<= 1;
            first_code[l] = code;
            first_idx[l] = idx;
            code += count[l];
            idx += count[l];
        }
        const unsigned long long nbits = get_u64(tab + 5ull * d);
        const unsigned char* bits = tab + 5ull * d + 8;
        unsigned long long pos = 0;
        int* o = out + block_first[b];
        for (unsigned i = 0; i < n; ++i) {
            unsigned c = 0;
            int l = 1;
            for (;; ++l) {
                if (l > max_len || pos >= nbits) {
                    atomicExch(err, 2);
                    return;
                }
                c = (c << 1) | ((bits[pos >> 3] >> (7 - (pos & 7))) & 1u);
                ++pos;
                const unsigned rel = c - first_code[l];
                if (c >= first_code[l] && rel < count[l]) {
                    const unsigned sym = get_u32(tab + 5ull * (first_idx[l] + rel));
                    o[i] = static_cast<int>((sym >> 1) ^ (~(sym & 1u) + 1u));  // unzigzag
                    break;
                }
            }
        }
    }
}

} // namespace

void huffman_decode_device(DevScratch& s, const unsigned char* payload, unsigned long long len,
                           const unsigned long long* block_off, const unsigned long long* block_first,
                           long long nb, int* codes_out) {
    cudaStream_t st = s.stream;
    if (nb == 0) return;
    auto* dp = static_cast<unsigned char*>(s.get("hd_payload", len));
    auto* doff = static_cast<unsigned long long*>(s.get("hd_off", 8 * nb));
    auto* dfirst = static_cast<unsigned long long*>(s.get("hd_first", 8 * nb));
    auto* err = static_cast<int*>(s.get("hd_err", 4));
    FFCZ_CUDA_CHECK(cudaMemcpyAsync(dp, payload, len, cudaMemcpyHostToDevice, st));
    FFCZ_CUDA_CHECK(cudaMemcpyAsync(doff, block_off, 8 * nb, cudaMemcpyHostToDevice, st));
    FFCZ_CUDA_CHECK(cudaMemcpyAsync(dfirst, block_first, 8 * nb, cudaMemcpyHostToDevice, st));
    FFCZ_CUDA_CHECK(cudaMemsetAsync(err, 0, 4, st));
    k_huff_decode<<<static_cast<unsigned>((nb + 31) / 32), 32, 0, st>>>(dp, doff, dfirst, nb,
                                                                        codes_out, err);
    FFCZ_LAUNCH_CHECK();
    int h = 0;
    FFCZ_CUDA_CHECK(cudaMemcpyAsync(&h, err, 4, cudaMemcpyDeviceToHost, st));
    FFCZ_CUDA_CHECK(cudaStreamSynchronize(st));
    if (h == 1) throw Error(kFormat, "huffman: bad code length or non-canonical table");
    if (h == 2) throw Error(kFormat, "huffman: invalid code");
}
} // namespace ffcz_gpu
