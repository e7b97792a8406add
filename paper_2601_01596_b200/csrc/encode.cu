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
#include <cstdio>
#include <chrono>
#include <cstdlib>
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

__global__ void k_zz_max(const int* __restrict__ codes, unsigned long long n, unsigned* zmax) {
    unsigned m = 0;
    for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < n;
         i += (unsigned long long)gridDim.x * blockDim.x)
        m = max(m, zz(codes[i]));
    for (int o = 16; o; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0 && m) atomicMax(zmax, m);
}

__global__ void k_keys32(const int* __restrict__ codes, unsigned long long n, int bs,
                         unsigned* keys) {
    for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < n;
         i += (unsigned long long)gridDim.x * blockDim.x)
        keys[i] = static_cast<unsigned>((i >> kBlockShift) << bs) | zz(codes[i]);
}

__global__ void k_widen_keys(const unsigned* __restrict__ k32, const int* nruns_p, int bs,
                             unsigned long long* ukeys) {
    const long long R = *nruns_p;
    const unsigned mask = bs >= 32 ? ~0u : ((1u << bs) - 1u);
    for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < R;
         r += (long long)gridDim.x * blockDim.x) {
        const unsigned k = k32[r];
        ukeys[r] = (static_cast<unsigned long long>(k >> bs) << 32) | (k & mask);
    }
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

// Leaf keys for the per-block (weight, symbol) order: block << 33 | count << 16 | rank, rank =
// the run's index inside its block (runs are symbol-ascending, so rank order = symbol order).
// count <= 65536 < 2^17, rank < 2^16.
__global__ void k_leaf_keys(const unsigned long long* __restrict__ ukeys,
                            const int* __restrict__ counts, const long long* __restrict__ run_start,
                            const int* nruns_p, unsigned long long* lkeys) {
    const long long R = *nruns_p;
    for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < R;
         r += (long long)gridDim.x * blockDim.x) {
        const unsigned long long b = ukeys[r] >> 32;
        const unsigned long long rank = static_cast<unsigned long long>(r - run_start[b]);
        lkeys[r] = (b << 33) | (static_cast<unsigned long long>(counts[r]) << 16) | rank;
    }
}

// One thread per block: Huffman code lengths exactly as the reference's heap computes them
// (huffman.cpp:74-120: repeatedly pair the two lightest subtrees, ties broken by the smallest
// symbol in the subtree), in O(d) with two queues instead of a heap:
//   * leaves arrive sorted by (weight, symbol) (the global leaf-key sort);
//   * internal nodes are created with non-decreasing weights, and a new node weighs more than
//     the minimum alive weight (w_a + w_b > w_b >= min), so when an internal node of weight w is
//     first needed (min alive weight == w) every internal node of weight w already exists and
//     they form one contiguous run at the queue head; that run is put in tie order once
//     (insertion sort of node ids; runs arrive nearly sorted);
//   * the head of each queue is then the (weight, tie)-minimum of its queue, so the pairing
//     sequence is the heap's.
// Then depths from parent links (parents are created after children), canonical order by a
// counting sort on length (symbol order kept inside a length) and canonical codes
// (huffman.cpp:122-154).  Scratch per block (offset r0 = run_start[b], d runs): iw / it / q of
// d - 1 internal nodes, par of 2d - 1 nodes.
__device__ void block_table_global(long long b, const unsigned long long* __restrict__ lkeys,
                                   const long long* __restrict__ run_start, unsigned* iw,
                                   unsigned* it, int* q, int* par, unsigned char* len_of_run,
                                   unsigned* code_of_run, int* canon) {
    {
        const long long r0 = run_start[b];
        const int d = static_cast<int>(run_start[b + 1] - r0);
        unsigned char* L = len_of_run + r0;
        if (d == 1) {
            L[0] = 1;  // huffman.cpp:76
        } else {
            const unsigned long long* LK = lkeys + r0;
            unsigned* W = iw + r0;
            unsigned* T = it + r0;
            int* Q = q + r0;
            int* P = par + 2 * r0;  // node ids: leaf = rank (0..d-1), internal k = d + k
            int li = 0, qh = 0, qn = 0, sorted_to = 0;
            auto pop = [&](unsigned& w, unsigned& t, int& id) {
                const bool have_l = li < d;
                if (qh < qn) {
                    const unsigned wi = W[Q[qh]];
                    const unsigned lw = have_l ? static_cast<unsigned>((LK[li] >> 16) & 0x1FFFFu) : 0;
                    if ((!have_l || lw >= wi) && sorted_to <= qh) {
                        int e = qh + 1;
                        while (e < qn && W[Q[e]] == wi) ++e;
                        for (int i = qh + 1; i < e; ++i) {  // insertion sort by tie
                            const int v = Q[i];
                            const unsigned tv = T[v];
                            int j = i - 1;
                            while (j >= qh && T[Q[j]] > tv) {
                                Q[j + 1] = Q[j];
                                --j;
                            }
                            Q[j + 1] = v;
                        }
                        sorted_to = e;
                    }
                    const int k = Q[qh];
                    bool take_internal = !have_l;
                    if (have_l) {
                        const unsigned lt = static_cast<unsigned>(LK[li] & 0xFFFFu);
                        take_internal = wi < lw || (wi == lw && T[k] < lt);
                    }
                    if (take_internal) {
                        w = wi;
                        t = T[k];
                        id = d + k;
                        ++qh;
                        return;
                    }
                }
                w = static_cast<unsigned>((LK[li] >> 16) & 0x1FFFFu);
                t = static_cast<unsigned>(LK[li] & 0xFFFFu);
                id = static_cast<int>(t);
                ++li;
            };
            for (int m = 0; m < d - 1; ++m) {
                unsigned wa, ta, wb, tb;
                int ia, ib;
                pop(wa, ta, ia);
                pop(wb, tb, ib);
                W[qn] = wa + wb;
                T[qn] = ta < tb ? ta : tb;
                Q[qn] = qn;
                P[ia] = d + qn;
                P[ib] = d + qn;
                ++qn;
            }
            // depths: root = internal qn-1; W reused as the depth of internal nodes
            W[qn - 1] = 0;
            for (int k = qn - 2; k >= 0; --k) W[k] = W[P[d + k] - d] + 1;
            for (int i = 0; i < d; ++i) L[i] = static_cast<unsigned char>(W[P[i] - d] + 1);
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


// One CTA per block (the common path): the same pairing sequence, produced in parallel batches.
// With w0 the smallest alive weight, every node created from now on weighs >= 2 w0, so all
// alive items lighter than 2 w0 are popped before any new node, in the merged (weight, tie)
// order of the two queues, and they pair up consecutively.  A batch therefore takes the first
// B such items (B even, <= kBatch; B = 2 when fewer exist: the two smallest always pair),
// finds each one's place by a merge-path search over the two queue heads staged in shared
// memory, and creates B/2 internal nodes at once (one thread per pair).  New nodes keep the
// internal queue in non-decreasing weight; its (weight, tie) order inside a batch's prefix is
// checked, and a block whose internal queue is ever out of tie order falls back to
// block_table_global (never observed; tests force that path).  An all-distinct 65,536-symbol
// block takes ~260 batches instead of 65,535 dependent steps.
// Depths then come from pointer jumping over the parent links (ping-pong buffers in global
// memory), the canonical order from a stable counting sort by length (per-thread chunks,
// per-length scans) and the canonical codes from first_code[len] + rank in the length.
constexpr int kBatch = 512;
constexpr int kTabThreads = 256;

__global__ void __launch_bounds__(kTabThreads)
k_block_tables_batch(const unsigned long long* __restrict__ lkeys,
                     const long long* __restrict__ run_start, long long nb, unsigned* iw,
                     unsigned* it, int* q, int* par, int* pj, unsigned char* len_of_run,
                     unsigned* code_of_run, int* canon, int mode) {
    __shared__ unsigned long long sl[kBatch], si[kBatch];  // (weight << 32 | tie) of the heads
    __shared__ int cntbuf[34 * kTabThreads];
    __shared__ int s_li, s_qh, s_qn, s_fallback, s_qnf, s_used;
    __shared__ int first_code[34], len_start[34], len_total[34];
    const int tid = threadIdx.x;
    for (long long b = blockIdx.x; b < nb; b += gridDim.x) {
        const long long r0 = run_start[b];
        const int d = static_cast<int>(run_start[b + 1] - r0);
        unsigned char* L = len_of_run + r0;
        if (d == 1) {
            if (tid == 0) {
                L[0] = 1;  // huffman.cpp:76
                canon[r0] = 0;
                code_of_run[r0] = 0;
            }
            __syncthreads();
            continue;
        }
        int* P = par + 2 * r0;  // node ids: leaf = rank, internal k = d + k
        unsigned* W = iw + r0;  // internal nodes: weight, tie
        unsigned* T = it + r0;
        const unsigned long long* LK = lkeys + r0;
        if (tid == 0) {
            s_li = 0;
            s_qh = 0;
            s_qn = 0;
            s_fallback = mode == 2;
        }
        __syncthreads();
        for (;;) {
            const int li = s_li, qh = s_qh, qn = s_qn;
            if ((d - li) + (qn - qh) <= 1 || s_fallback) break;
            const int nL = min(kBatch, d - li), nI = min(kBatch, qn - qh);
            for (int t = tid; t < kBatch; t += kTabThreads) {
                if (t < nL) {
                    const unsigned long long k = LK[li + t];
                    sl[t] = (((k >> 16) & 0x1FFFFull) << 32) | (k & 0xFFFFull);
                }
                if (t < nI) si[t] = (static_cast<unsigned long long>(W[qh + t]) << 32) | T[qh + t];
            }
            __syncthreads();
            const unsigned long long w0 =
                min(nL ? sl[0] >> 32 : ~0ull, nI ? si[0] >> 32 : ~0ull);
            const unsigned long long lim = (2 * w0) << 32;  // keys below: weight < 2 w0
            auto count_below = [&](const unsigned long long* a, int n) {
                int lo = 0, hi = n;
                while (lo < hi) {
                    const int mid = (lo + hi) >> 1;
                    if (a[mid] < lim) lo = mid + 1;
                    else hi = mid;
                }
                return lo;
            };
            const int n_l = count_below(sl, nL), n_i = count_below(si, nI);
            int B = min(n_l + n_i, kBatch) & ~1;
            if (B < 2) B = 2;
            // the internal heads this batch may consume must be in (weight, tie) order
            bool bad = false;
            for (int t = tid + 1; t < min(B + 1, nI); t += kTabThreads)
                if (!(si[t - 1] < si[t])) bad = true;
            if (__syncthreads_or(bad)) {
                if (tid == 0) s_fallback = 1;
                __syncthreads();
                break;
            }
            // merge path: number of leaves among the first p merged items
            auto split = [&](int p) {
                int lo = max(0, p - nI), hi = min(p, nL);
                while (lo < hi) {
                    const int mid = (lo + hi) >> 1;
                    if (sl[mid] < si[p - mid - 1]) lo = mid + 1;
                    else hi = mid;
                }
                return lo;
            };
            auto item = [&](int p, unsigned long long& key, int& id) {
                const int i = split(p);
                const bool leaf = i < nL && (p - i >= nI || sl[i] < si[p - i]);
                if (leaf) {
                    key = sl[i];
                    id = static_cast<int>(key & 0xFFFFu);
                } else {
                    key = si[p - i];
                    id = d + qh + (p - i);
                }
            };
            if (tid < B / 2) {
                unsigned long long ka, kb;
                int ia, ib;
                item(2 * tid, ka, ia);
                item(2 * tid + 1, kb, ib);
                const int k = qn + tid;
                W[k] = static_cast<unsigned>((ka >> 32) + (kb >> 32));
                T[k] = static_cast<unsigned>(min(ka & 0xFFFFFFFFull, kb & 0xFFFFFFFFull));
                P[ia] = d + k;
                P[ib] = d + k;
            }
            if (tid == 0) s_used = split(B);
            __syncthreads();
            if (tid == 0) {
                s_li = li + s_used;
                s_qh = qh + (B - s_used);
                s_qn = qn + B / 2;
            }
            __syncthreads();
        }
        if (tid == 0) s_qnf = s_qn;
        __syncthreads();
        if (s_fallback) {
            if (tid == 0)
                block_table_global(b, lkeys, run_start, iw, it, q, par, len_of_run, code_of_run,
                                   canon);
            __syncthreads();
            continue;
        }
        const int s_qn_final = s_qnf;
    // depths of the internal nodes by pointer jumping (root = qn - 1)
        const int qn = s_qn_final;
        int* dep0 = reinterpret_cast<int*>(iw + r0);
        int* anc0 = reinterpret_cast<int*>(it + r0);
        int* dep1 = q + r0;
        int* anc1 = pj + r0;
        for (int k = tid; k < qn; k += kTabThreads) {
            const bool root = k == qn - 1;
            dep0[k] = root ? 0 : 1;
            anc0[k] = root ? k : P[d + k] - d;
        }
        __syncthreads();
        for (int round = 0; round < 6; ++round) {  // depth <= 32 < 2^6
            for (int k = tid; k < qn; k += kTabThreads) {
                const int a = anc0[k];
                dep1[k] = dep0[k] + (a != k ? dep0[a] : 0);
                anc1[k] = anc0[a];
            }
            __syncthreads();
            int* t0 = dep0; dep0 = dep1; dep1 = t0;
            int* t1 = anc0; anc0 = anc1; anc1 = t1;
        }
        for (int i = tid; i < d; i += kTabThreads) L[i] = static_cast<unsigned char>(dep0[P[i] - d] + 1);
        __syncthreads();
        // canonical order: stable counting sort of the symbol-ascending runs by length
        int* cnt = cntbuf;  // [34][kTabThreads]
        const int chunk = (d + kTabThreads - 1) / kTabThreads;
        const int i0 = tid * chunk, i1 = min(d, i0 + chunk);
        for (int l = 0; l < 34; ++l) cnt[l * kTabThreads + tid] = 0;
        for (int i = i0; i < i1; ++i) ++cnt[L[i] * kTabThreads + tid];
        __syncthreads();
        if (tid < 34) {  // per length: exclusive scan over threads, total
            int acc = 0;
            for (int t = 0; t < kTabThreads; ++t) {
                const int v = cnt[tid * kTabThreads + t];
                cnt[tid * kTabThreads + t] = acc;
                acc += v;
            }
            len_total[tid] = acc;
        }
        __syncthreads();
        if (tid == 0) {
            int acc = 0;
            unsigned code = 0;
            for (int l = 0; l < 34; ++l) {
                len_start[l] = acc;
                acc += len_total[l];
                first_code[l] = static_cast<int>(code);  // huffman.cpp:128-138
                code = (code + (l ? len_total[l] : 0)) << 1;
            }
        }
        __syncthreads();
        int* cn = canon + r0;
        for (int i = i0; i < i1; ++i) {
            const int l = L[i];
            const int rank = cnt[l * kTabThreads + tid]++;
            cn[len_start[l] + rank] = i;
            code_of_run[r0 + i] = static_cast<unsigned>(first_code[l]) + static_cast<unsigned>(rank);
        }
        __syncthreads();
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

// FFCZ_HUFFMAN_TABLES=global: every block through block_table_global (test hook for the
// fallback path)
int table_mode() {
    const char* e = std::getenv("FFCZ_HUFFMAN_TABLES");
    if (!e) return 0;
    return std::strcmp(e, "global") == 0 ? 2 : 0;
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
    // FFCZ_DEBUG_TIMING=1: host timestamps of the encoder's steps on stderr (synchronises)
    static const bool dbg_on = std::getenv("FFCZ_DEBUG_TIMING") != nullptr;
    const auto t_start = std::chrono::steady_clock::now();
    auto mark = [&](const char* what) {
        if (!dbg_on) return;
        cudaStreamSynchronize(st);
        std::fprintf(stderr, "[ffcz] huffman: %-20s %9.3f ms\n", what,
                     std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() -
                                                               t_start).count());
    };
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
    // the widest zigzag symbol decides the key layout: when block and symbol bits fit 32 bits
    // the sort and run-length run on 32-bit keys (block << bs | zz: half the traffic and 4 radix
    // passes instead of 6 at 1024^3), widened to (block << 32 | zz) for the later steps
    auto* zmax = static_cast<unsigned*>(s.get("huf_zmax", 4));
    FFCZ_CUDA_CHECK(cudaMemsetAsync(zmax, 0, 4, st));
    k_zz_max<<<grid_n(n), 256, 0, st>>>(codes, n, zmax);
    FFCZ_LAUNCH_CHECK();
    unsigned h_zmax = 0;
    FFCZ_CUDA_CHECK(cudaMemcpyAsync(&h_zmax, zmax, 4, cudaMemcpyDeviceToHost, st));
    FFCZ_CUDA_CHECK(cudaStreamSynchronize(st));
    int bs = 1, bb = 0;
    while (bs < 32 && (1ull << bs) <= h_zmax) ++bs;
    while ((1ll << bb) < nb) ++bb;
    const bool narrow = bs + bb <= 32;
    if (narrow) {
        auto* k32 = reinterpret_cast<unsigned*>(keys);
        auto* s32 = k32 + n;
        auto* u32k = reinterpret_cast<unsigned*>(skeys);
        k_keys32<<<grid_n(n), 256, 0, st>>>(codes, n, bs, k32);
        FFCZ_LAUNCH_CHECK();
        cub_call(s, "huf_tmp_sort32", [&](void* t, size_t& b) {
            return cub::DeviceRadixSort::SortKeys(t, b, k32, s32, static_cast<int64_t>(n), 0,
                                                  bs + bb, st);
        });
        cub_call(s, "huf_tmp_rle32", [&](void* t, size_t& b) {
            return cub::DeviceRunLengthEncode::Encode(t, b, s32, u32k, counts, nruns,
                                                      static_cast<int64_t>(n), st);
        });
        k_widen_keys<<<grid_n(n), 256, 0, st>>>(u32k, nruns, bs, ukeys);
        FFCZ_LAUNCH_CHECK();
    } else {
        k_keys<<<grid_n(n), 256, 0, st>>>(codes, n, keys);
        FFCZ_LAUNCH_CHECK();
        cub_call(s, "huf_tmp_sort", [&](void* t, size_t& b) {
            return cub::DeviceRadixSort::SortKeys(t, b, keys, skeys, static_cast<int64_t>(n), 0,
                                                  32 + bb, st);
        });
        cub_call(s, "huf_tmp_rle", [&](void* t, size_t& b) {
            return cub::DeviceRunLengthEncode::Encode(t, b, skeys, ukeys, counts, nruns,
                                                      static_cast<int64_t>(n), st);
        });
    }
    mark("keys sorted, runs");
    int h_nruns = 0;
    FFCZ_CUDA_CHECK(cudaMemcpyAsync(&h_nruns, nruns, 4, cudaMemcpyDeviceToHost, st));
    FFCZ_CUDA_CHECK(cudaStreamSynchronize(st));
    const long long R = h_nruns;
    auto* run_start = static_cast<long long*>(s.get("huf_run_start", 8 * (nb + 1)));
    k_block_runs<<<grid_n(nb + 1), 256, 0, st>>>(ukeys, nruns, nb, run_start);
    // leaves of every block in (weight, symbol) order: one radix sort of the run keys
    auto* lkeys = static_cast<unsigned long long*>(s.get("huf_lkeys", 8 * R));
    auto* lkeys_s = static_cast<unsigned long long*>(s.get("huf_lkeys_s", 8 * R));
    k_leaf_keys<<<grid_n(R), 256, 0, st>>>(ukeys, counts, run_start, nruns, lkeys);
    FFCZ_LAUNCH_CHECK();
    int lend = 33;
    while ((1ll << (lend - 33)) < nb) ++lend;
    // sort on (block, count) only: the radix sort is stable and the runs arrive in (block,
    // symbol) order, so the rank bits [0, 16) ride along already in tie order (6 -> 4 passes)
    cub_call(s, "huf_tmp_sort2", [&](void* t, size_t& b) {
        return cub::DeviceRadixSort::SortKeys(t, b, lkeys, lkeys_s, static_cast<int64_t>(R), 16,
                                              lend, st);
    });
    auto* iw = static_cast<unsigned*>(s.get("huf_iw", 4 * R));
    auto* it = static_cast<unsigned*>(s.get("huf_it", 4 * R));
    auto* iq = static_cast<int*>(s.get("huf_iq", 4 * R));
    auto* par = static_cast<int*>(s.get("huf_par", 8 * R));
    auto* len_of_run = static_cast<unsigned char*>(s.get("huf_len", R));
    auto* code_of_run = static_cast<unsigned*>(s.get("huf_code", 4 * R));
    auto* canon = static_cast<int*>(s.get("huf_canon", 4 * R));
    auto* pj = static_cast<int*>(s.get("huf_pj", 4 * R));
    int per_sm = 0;
    FFCZ_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_block_tables_batch,
                                                                  kTabThreads, 0));
    const long long grid = std::min<long long>(nb, 148ll * std::max(1, per_sm));
    k_block_tables_batch<<<static_cast<unsigned>(grid), kTabThreads, 0, st>>>(
        lkeys_s, run_start, nb, iw, it, iq, par, pj, len_of_run, code_of_run, canon,
        table_mode());
    FFCZ_LAUNCH_CHECK();
    mark("code tables");
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
    mark("symbol codes, scans");
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
    mark("bits packed, written");
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

// One thread per block: the canonical decode of huffman.cpp:205-243, by limits instead of bit by
// bit: with the next 32 bits of the stream as a left-aligned window w, the code length is the
// smallest l with w < lim[l] (lim[l] = first code after the length-l codes, left-aligned), and
// the symbol is table[first_idx[l] + (w >> (32 - l)) - first_code[l]].  The stream is read
// through a 64-bit big-endian bit buffer refilled a byte at a time.
__global__ void k_huff_decode(const unsigned char* __restrict__ payload,
                              const unsigned long long* __restrict__ block_off,
                              const unsigned long long* __restrict__ block_first, long long nb,
                              int* out, int* err) {
    for (long long b = blockIdx.x * (long long)blockDim.x + threadIdx.x; b < nb;
         b += (long long)gridDim.x * blockDim.x) {
        const unsigned char* p = payload + block_off[b];
        const unsigned n = get_u32(p), d = get_u32(p + 4);
        const unsigned char* tab = p + 8;
        unsigned count[33];
        for (int l = 0; l <= 32; ++l) count[l] = 0;
        int max_len = 0, min_len = 33;
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
            min_len = len < static_cast<unsigned>(min_len) ? len : min_len;
        }
        if (bad) {
            atomicExch(err, 1);
            continue;
        }
        // canonical first codes / indices (huffman.cpp:205-215) and left-aligned limits
        unsigned first_code[33], first_idx[33];
        unsigned long long lim[33];
        unsigned code = 0, idx = 0;
        for (int l = 1; l <= 32; ++l) {
            code <<= 1;
            first_code[l] = code;
            first_idx[l] = idx;
            code += count[l];
            idx += count[l];
            lim[l] = static_cast<unsigned long long>(code) << (32 - l);  // may be 2^32
        }
        const unsigned long long nbits = get_u64(tab + 5ull * d);
        const unsigned char* bits = tab + 5ull * d + 8;
        const unsigned long long nbytes = (nbits + 7) / 8;
        unsigned long long buf = 0, pos = 0, byte_at = 0;
        int have = 0;  // valid bits in buf (left-aligned at bit 63)
        int* o = out + block_first[b];
        bool fail = false;
        for (unsigned i = 0; i < n && !fail; ++i) {
            while (have <= 56) {
                const unsigned long long v = byte_at < nbytes ? bits[byte_at] : 0;
                ++byte_at;
                buf |= v << (56 - have);
                have += 8;
            }
            const unsigned long long w = buf >> 32;  // next 32 bits
            int l = min_len;
            while (l <= max_len && w >= lim[l]) ++l;
            if (l > max_len || pos + static_cast<unsigned long long>(l) > nbits) {
                fail = true;
                break;
            }
            const unsigned c = static_cast<unsigned>(w >> (32 - l));
            const unsigned sym = get_u32(tab + 5ull * (first_idx[l] + (c - first_code[l])));
            o[i] = static_cast<int>((sym >> 1) ^ (~(sym & 1u) + 1u));  // unzigzag
            buf <<= l;
            have -= l;
            pos += l;
        }
        if (fail) atomicExch(err, 2);
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
