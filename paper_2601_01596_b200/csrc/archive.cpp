// Host-side .ffcz archive writer (the zlib_level 0..9 modes; the default archive is assembled
// from device-encoded streams, archive_dev.cu).  Byte layout follows
// /root/reference/proj/docs/FORMAT.md and the reference writer (archive.cpp:73-135,
// streams.cpp:21-55, huffman.cpp:156-251) so that the reference's read_archive decodes it and,
// with zlib level 9 and identical edits, the bytes are identical.  The edits themselves follow the
// engine's defaults (decoder-view escape repair, F rebuilt at the gate: INTEGRATION.md §4), which
// can differ from the reference's where FP64 round-off straddles a bound; the per-call option
// flags FFCZ_REPAIR_REFERENCE_ORDER / FFCZ_F_ACCUMULATE select the reference's order.
#include "archive.hpp"

#include <zlib.h>

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <exception>
#include <future>
#include <thread>
#include <queue>
#include <stdexcept>
#include <string>

namespace ffcz_host {

namespace {

template <class T>
void put(std::vector<std::uint8_t>& out, T v) {
    std::uint8_t b[sizeof(T)];
    std::memcpy(b, &v, sizeof(T));
    out.insert(out.end(), b, b + sizeof(T));
}

constexpr std::size_t kBlockSymbols = std::size_t(1) << 16;  // huffman.hpp:13

// Code lengths from repeatedly pairing the two lightest subtrees, ordered by
// (weight, smallest contained symbol) — the reference's deterministic tie-break
// (huffman.cpp:74-120).  (weight, tiebreak) pairs are unique, so the pairing sequence and hence
// every depth is implementation-independent.
std::vector<std::uint8_t> code_lengths(const std::vector<std::uint32_t>& syms,
                                       const std::vector<std::uint64_t>& w) {
    const std::size_t n = syms.size();
    if (n == 1) return {1};
    struct Node {
        std::uint64_t weight;
        std::uint32_t tie;
        int left, right;
    };
    std::vector<Node> nodes;
    nodes.reserve(2 * n);
    using Key = std::pair<std::pair<std::uint64_t, std::uint32_t>, int>;
    std::priority_queue<Key, std::vector<Key>, std::greater<Key>> heap;
    for (std::size_t i = 0; i < n; ++i) {
        nodes.push_back({w[i], syms[i], -1, -1});
        heap.push({{w[i], syms[i]}, static_cast<int>(i)});
    }
    while (heap.size() > 1) {
        const int a = heap.top().second;
        heap.pop();
        const int b = heap.top().second;
        heap.pop();
        nodes.push_back({nodes[a].weight + nodes[b].weight, std::min(nodes[a].tie, nodes[b].tie), a, b});
        const int id = static_cast<int>(nodes.size()) - 1;
        heap.push({{nodes[id].weight, nodes[id].tie}, id});
    }
    std::vector<std::uint8_t> len(n, 0);
    std::vector<std::pair<int, int>> stack{{heap.top().second, 0}};
    while (!stack.empty()) {
        auto [id, d] = stack.back();
        stack.pop_back();
        if (nodes[id].left < 0) {
            len[id] = static_cast<std::uint8_t>(d);
        } else {
            stack.push_back({nodes[id].left, d + 1});
            stack.push_back({nodes[id].right, d + 1});
        }
    }
    return len;
}

struct BitSink {
    std::vector<std::uint8_t>& out;
    std::uint64_t acc = 0;  // pending bits, MSB-first
    int nacc = 0;
    std::uint64_t total = 0;
    void put(std::uint32_t code, int len) {
        total += static_cast<std::uint64_t>(len);
        // flush whole bytes while keeping <= 56 pending bits
        acc = (acc << len) | (len == 32 ? code : (code & ((1u << len) - 1u)));
        nacc += len;
        while (nacc >= 8) {
            nacc -= 8;
            out.push_back(static_cast<std::uint8_t>(acc >> nacc));
        }
        acc &= (nacc ? ((std::uint64_t(1) << nacc) - 1) : 0);
    }
    void flush() {
        if (nacc > 0) out.push_back(static_cast<std::uint8_t>(acc << (8 - nacc)));
        acc = 0;
        nacc = 0;
    }
};

void encode_block(std::vector<std::uint8_t>& out, const std::uint32_t* data, std::size_t n) {
    std::vector<std::uint32_t> sorted(data, data + n);
    std::sort(sorted.begin(), sorted.end());
    std::vector<std::uint32_t> syms;
    std::vector<std::uint64_t> counts;
    for (std::size_t i = 0; i < n;) {
        std::size_t j = i;
        while (j < n && sorted[j] == sorted[i]) ++j;
        syms.push_back(sorted[i]);
        counts.push_back(j - i);
        i = j;
    }
    const std::vector<std::uint8_t> lens = code_lengths(syms, counts);
    // canonical order (length, symbol) and codes (huffman.cpp:124-154)
    std::vector<std::size_t> order(syms.size());
    for (std::size_t i = 0; i < order.size(); ++i) order[i] = i;
    std::sort(order.begin(), order.end(), [&](std::size_t a, std::size_t b) {
        return lens[a] != lens[b] ? lens[a] < lens[b] : syms[a] < syms[b];
    });
    std::vector<std::uint32_t> code_of(syms.size());
    std::uint32_t code = 0;
    int prev = 0;
    for (std::size_t r = 0; r < order.size(); ++r) {
        const std::size_t i = order[r];
        code <<= (lens[i] - prev);
        code_of[i] = code++;
        prev = lens[i];
    }
    put<std::uint32_t>(out, static_cast<std::uint32_t>(n));
    put<std::uint32_t>(out, static_cast<std::uint32_t>(syms.size()));
    for (std::size_t i : order) {
        put<std::uint32_t>(out, syms[i]);
        put<std::uint8_t>(out, lens[i]);
    }
    const std::size_t nbits_pos = out.size();
    put<std::uint64_t>(out, 0);
    BitSink bs{out};
    for (std::size_t i = 0; i < n; ++i) {
        const std::size_t s = std::lower_bound(syms.begin(), syms.end(), data[i]) - syms.begin();
        bs.put(code_of[s], lens[s]);
    }
    bs.flush();
    std::memcpy(out.data() + nbits_pos, &bs.total, sizeof(std::uint64_t));
}

} // namespace

#if defined(__x86_64__)
// SSE4.2 `crc32` computes exactly CRC-32C (Castagnoli, reflected 0x82F63B78): 8 bytes per
// instruction instead of one table lookup per byte (the 2 GB per-component Delta header of a
// 512^3 config-2 archive: ~0.3 s instead of ~4 s).
__attribute__((target("sse4.2"))) static std::uint32_t crc32c_sse42(const std::uint8_t* p,
                                                                    std::size_t n) {
    std::uint64_t c = 0xFFFFFFFFu;
    while (n && (reinterpret_cast<std::uintptr_t>(p) & 7u)) {
        c = __builtin_ia32_crc32qi(static_cast<std::uint32_t>(c), *p++);
        --n;
    }
    while (n >= 8) {
        std::uint64_t v;
        std::memcpy(&v, p, 8);
        c = __builtin_ia32_crc32di(c, v);
        p += 8;
        n -= 8;
    }
    while (n--) c = __builtin_ia32_crc32qi(static_cast<std::uint32_t>(c), *p++);
    return static_cast<std::uint32_t>(c) ^ 0xFFFFFFFFu;
}
#endif

std::uint32_t crc32c(const std::uint8_t* data, std::size_t len) {
#if defined(__x86_64__)
    static const bool hw = __builtin_cpu_supports("sse4.2");
    if (hw) return crc32c_sse42(data, len);
#endif
    static std::uint32_t table[256];
    static bool init = [] {
        for (std::uint32_t i = 0; i < 256; ++i) {
            std::uint32_t c = i;
            for (int j = 0; j < 8; ++j) c = (c >> 1) ^ (0x82F63B78u & (0u - (c & 1u)));
            table[i] = c;
        }
        return true;
    }();
    (void)init;
    std::uint32_t crc = 0xFFFFFFFFu;
    for (std::size_t i = 0; i < len; ++i) crc = (crc >> 8) ^ table[(crc ^ data[i]) & 0xFFu];
    return crc ^ 0xFFFFFFFFu;
}

int host_threads() {
    const unsigned hw = std::thread::hardware_concurrency();
    return static_cast<int>(std::clamp(hw ? hw : 1u, 1u, 16u));
}

std::uint32_t crc32c_combine(std::uint32_t crc1, std::uint32_t crc2, std::uint64_t len2);

std::uint32_t crc32c_threads(const std::uint8_t* p, std::uint64_t n) {
    const int T = n < (std::uint64_t(64) << 20) ? 1 : host_threads();
    if (T == 1) return crc32c(p, n);
    std::vector<std::uint32_t> part(T);
    std::vector<std::uint64_t> lo(T + 1);
    for (int t = 0; t <= T; ++t) lo[t] = n * t / T;
    std::vector<std::thread> th;
    for (int t = 0; t < T; ++t)
        th.emplace_back([&, t] { part[t] = crc32c(p + lo[t], lo[t + 1] - lo[t]); });
    for (auto& x : th) x.join();
    std::uint32_t c = part[0];
    for (int t = 1; t < T; ++t) c = crc32c_combine(c, part[t], lo[t + 1] - lo[t]);
    return c;
}

std::uint32_t zigzag(std::int32_t v) {
    return (static_cast<std::uint32_t>(v) << 1) ^ static_cast<std::uint32_t>(v >> 31);
}

std::vector<std::uint8_t> huffman_encode(const std::uint32_t* symbols, std::size_t n) {
    std::vector<std::uint8_t> out;
    put<std::uint64_t>(out, n);
    for (std::size_t s = 0; s < n; s += kBlockSymbols)
        encode_block(out, symbols + s, std::min(kBlockSymbols, n - s));
    return out;
}

std::vector<std::uint8_t> outer_compress(const std::uint8_t* raw, std::size_t n, int level) {
    uLongf bound = compressBound(static_cast<uLong>(n));
    std::vector<std::uint8_t> out(sizeof(std::uint64_t) + bound);
    const std::uint64_t raw_size = n;
    std::memcpy(out.data(), &raw_size, sizeof(raw_size));
    static const Bytef empty = 0;
    const int rc = compress2(out.data() + sizeof(raw_size), &bound, n ? raw : &empty,
                             static_cast<uLong>(n), level);
    if (rc != Z_OK) throw std::runtime_error("outer_compress failed: zlib rc " + std::to_string(rc));
    out.resize(sizeof(raw_size) + bound);
    return out;
}

std::vector<std::uint8_t> write_archive(const ArchiveInput& in) {
    std::uint64_t N = 1;
    for (int a = 0; a < in.ndim; ++a) N *= in.dims[a];

    auto index_stream = [&](const std::int32_t* codes, std::size_t n) {
        std::vector<std::uint32_t> sym(n);
        for (std::size_t i = 0; i < n; ++i) sym[i] = zigzag(codes[i]);
        const std::vector<std::uint8_t> h = huffman_encode(sym.data(), n);
        return outer_compress(h.data(), h.size(), in.zlib_level);
    };
    const auto sf = outer_compress(in.spatial_flags, in.spatial_flag_bytes, in.zlib_level);
    const auto ff = outer_compress(in.frequency_flags, in.frequency_flag_bytes, in.zlib_level);
    const auto si = in.spatial_payload
                        ? outer_compress(in.spatial_payload, in.spatial_payload_len, in.zlib_level)
                        : index_stream(in.spatial_codes, in.n_spatial);
    const auto fi = in.frequency_payload
                        ? outer_compress(in.frequency_payload, in.frequency_payload_len, in.zlib_level)
                        : index_stream(in.frequency_codes, 2 * in.n_frequency);

    std::vector<std::uint8_t> w;
    w.reserve(128 + 8 * (in.spatial_per_point ? N : 1) + 16 * (in.freq_per_component ? N : 1) +
              sf.size() + ff.size() + si.size() + fi.size() + 24 * in.n_escapes);
    const char magic[4] = {'F', 'F', 'C', 'Z'};
    w.insert(w.end(), magic, magic + 4);
    put<std::uint16_t>(w, 1);
    put<std::uint8_t>(w, static_cast<std::uint8_t>(in.ndim));
    for (int a = 0; a < in.ndim; ++a) put<std::uint64_t>(w, in.dims[a]);
    put<std::uint8_t>(w, static_cast<std::uint8_t>(in.precision));
    std::uint8_t tags = 0;
    if (in.spatial_per_point) tags |= 1u;
    if (in.freq_per_component) tags |= 2u;
    if (in.converged) tags |= 4u;
    put<std::uint8_t>(w, tags);
    auto put_doubles = [&](const double* v, std::uint64_t n) {  // one copy, no zero-fill
        const auto* b = reinterpret_cast<const std::uint8_t*>(v);
        w.insert(w.end(), b, b + n * sizeof(double));
    };
    if (in.spatial_per_point) put_doubles(in.spatial_values, N);
    else put<double>(w, in.spatial_global);
    if (in.freq_per_component) {
        put_doubles(in.freq_re, N);
        put_doubles(in.freq_im, N);
    } else {
        put<double>(w, in.freq_global);
    }
    put<std::uint8_t>(w, static_cast<std::uint8_t>(in.m));
    put<std::uint64_t>(w, in.n_spatial);
    put<std::uint64_t>(w, in.n_frequency);
    put<std::uint64_t>(w, sf.size());
    put<std::uint64_t>(w, ff.size());
    put<std::uint64_t>(w, si.size());
    put<std::uint64_t>(w, fi.size());
    put<std::uint64_t>(w, in.n_escapes);
    put<std::uint32_t>(w, crc32c(w.data(), w.size()));
    w.insert(w.end(), sf.begin(), sf.end());
    w.insert(w.end(), ff.begin(), ff.end());
    w.insert(w.end(), si.begin(), si.end());
    w.insert(w.end(), fi.begin(), fi.end());
    for (std::uint64_t i = 0; i < in.n_escapes; ++i) {
        const EscapeRec& e = in.escapes[i];
        put<std::uint64_t>(w, e.index | (e.frequency ? (std::uint64_t(1) << 63) : 0));
        put<double>(w, e.re);
        if (e.frequency) put<double>(w, e.im);
    }
    return w;
}


namespace {

struct ArchiveError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

struct Reader {
    const std::uint8_t* p;
    std::size_t n, off = 0;
    template <class T> T pod() {
        if (off + sizeof(T) > n) throw ArchiveError("read_archive: truncated archive");
        T v;
        std::memcpy(&v, p + off, sizeof(T));
        off += sizeof(T);
        return v;
    }
    const std::uint8_t* take(std::size_t k) {
        if (off + k > n) throw ArchiveError("read_archive: truncated archive");
        const std::uint8_t* q = p + off;
        off += k;
        return q;
    }
};

std::vector<std::uint8_t> outer_decompress(const std::uint8_t* frame, std::size_t len) {
    if (len < sizeof(std::uint64_t)) throw ArchiveError("outer frame truncated");
    std::uint64_t raw = 0;
    std::memcpy(&raw, frame, sizeof(raw));
    std::vector<std::uint8_t> out(raw);
    if (raw == 0) return out;
    uLongf got = static_cast<uLongf>(raw);
    const int rc = uncompress(out.data(), &got, frame + sizeof(raw),
                              static_cast<uLong>(len - sizeof(raw)));
    if (rc != Z_OK || got != raw) throw ArchiveError("outer_decompress failed: corrupt frame");
    return out;
}

} // namespace

ParsedArchive parse_archive(const std::uint8_t* bytes, std::size_t len) {
    Reader r{bytes, len};
    ParsedArchive a;
    const std::uint8_t* magic = r.take(4);
    if (std::memcmp(magic, "FFCZ", 4) != 0) throw ArchiveError("read_archive: bad magic");
    if (r.pod<std::uint16_t>() != 1) throw ArchiveError("read_archive: unsupported version");
    a.ndim = r.pod<std::uint8_t>();
    if (a.ndim < 1 || a.ndim > 3) throw ArchiveError("read_archive: bad dimensionality");
    std::uint64_t N = 1;
    for (int i = 0; i < a.ndim; ++i) {
        a.dims[i] = r.pod<std::uint64_t>();
        if (a.dims[i] == 0) throw ArchiveError("read_archive: zero extent");
        N *= a.dims[i];
    }
    const std::uint8_t prec = r.pod<std::uint8_t>();
    if (prec > 1) throw ArchiveError("read_archive: bad precision tag");
    a.precision = prec;
    const std::uint8_t tags = r.pod<std::uint8_t>();
    a.spatial_per_point = tags & 1u;
    a.freq_per_component = tags & 2u;
    a.converged = tags & 4u;
    if (a.spatial_per_point) a.spatial_values = r.take(8 * N);
    else a.spatial_global = r.pod<double>();
    if (a.freq_per_component) {
        a.freq_re = r.take(8 * N);
        a.freq_im = r.take(8 * N);
    } else {
        a.freq_global = r.pod<double>();
    }
    a.m = r.pod<std::uint8_t>();
    if (a.m < 1 || a.m > 24) throw ArchiveError("read_archive: bad quantization width");
    a.n_spatial = r.pod<std::uint64_t>();
    a.n_frequency = r.pod<std::uint64_t>();
    const std::uint64_t lsf = r.pod<std::uint64_t>(), lff = r.pod<std::uint64_t>();
    const std::uint64_t lsi = r.pod<std::uint64_t>(), lfi = r.pod<std::uint64_t>();
    const std::uint64_t nesc = r.pod<std::uint64_t>();
    const std::size_t header_len = r.off;
    // (the bound arrays make the header up to 3 x 8 N bytes: CRC on host threads)
    if (crc32c_threads(bytes, header_len) != r.pod<std::uint32_t>())
        throw ArchiveError("read_archive: header checksum mismatch");
    const std::uint8_t* sf = r.take(lsf);
    const std::uint8_t* ff = r.take(lff);
    const std::uint8_t* si = r.take(lsi);
    const std::uint8_t* fi = r.take(lfi);
    // the four outer stages inflate concurrently
    auto fut_si = std::async(std::launch::async, [&] { return outer_decompress(si, lsi); });
    auto fut_fi = std::async(std::launch::async, [&] { return outer_decompress(fi, lfi); });
    auto fut_ff = std::async(std::launch::async, [&] { return outer_decompress(ff, lff); });
    std::exception_ptr err;
    try {
        a.spatial_flags = outer_decompress(sf, lsf);
    } catch (...) {
        err = std::current_exception();
    }
    auto get = [&](auto& fut, std::vector<std::uint8_t>& dst) {
        try {
            dst = fut.get();
        } catch (...) {
            if (!err) err = std::current_exception();
        }
    };
    get(fut_ff, a.frequency_flags);
    get(fut_si, a.spatial_payload);
    get(fut_fi, a.frequency_payload);
    if (err) std::rethrow_exception(err);
    std::uint64_t Nh = N / a.dims[a.ndim - 1] * (a.dims[a.ndim - 1] / 2 + 1);
    if (a.spatial_flags.size() != (N + 7) / 8 || a.frequency_flags.size() != (Nh + 7) / 8)
        throw ArchiveError("decode_streams: flag payload length mismatch");
    a.escapes.resize(nesc);
    for (auto& e : a.escapes) {
        const std::uint64_t packed = r.pod<std::uint64_t>();
        e.frequency = packed >> 63;
        e.index = packed & ~(std::uint64_t(1) << 63);
        e.re = r.pod<double>();
        e.im = e.frequency ? r.pod<double>() : 0.0;
        if (e.index >= (e.frequency ? Nh : N))
            throw ArchiveError("read_archive: escape index out of range");
    }
    if (r.off != len) throw ArchiveError("read_archive: trailing bytes");
    return a;
}

std::uint64_t huffman_blocks(const std::vector<std::uint8_t>& payload,
                             std::vector<std::uint64_t>& block_off,
                             std::vector<std::uint64_t>& block_first) {
    Reader r{payload.data(), payload.size()};
    const std::uint64_t total = r.pod<std::uint64_t>();
    std::uint64_t done = 0;
    while (done < total) {
        block_off.push_back(r.off);
        block_first.push_back(done);
        const std::uint32_t n = r.pod<std::uint32_t>();
        const std::uint32_t d = r.pod<std::uint32_t>();
        if (d == 0 || d > n) throw ArchiveError("huffman: bad table size");
        r.take(5ull * d);
        const std::uint64_t nbits = r.pod<std::uint64_t>();
        r.take((nbits + 7) / 8);
        done += n;
    }
    if (done != total || r.off != payload.size())
        throw ArchiveError("huffman: stream length mismatch");
    return total;
}
} // namespace ffcz_host
