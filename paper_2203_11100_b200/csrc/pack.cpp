// pack.cpp -- see pack.hpp for the layout.
#include "pack.hpp"

#include <algorithm>
#include <atomic>
#include <cstring>
#include <numeric>
#include <thread>

namespace swb {
namespace {

struct Key {
    uint32_t len;
    uint32_t idx;
};

// (length desc, db_index asc): the order both pools are stored in.
inline bool longer_first(const Key& a, const Key& b) {
    return a.len != b.len ? a.len > b.len : a.idx < b.idx;
}

// Snake deal: positions 0..G-1 go to shards 0..G-1, the next G positions to G-1..0, and so on.
inline uint32_t snake(uint64_t pos, uint32_t shards) {
    const uint64_t round = pos / shards;
    const uint32_t k = static_cast<uint32_t>(pos % shards);
    return (round & 1) ? shards - 1 - k : k;
}

void sorted_pools(const SeqSource& src, uint64_t threshold, std::vector<Key>& shorts,
                  std::vector<Key>& longs) {
    shorts.clear();
    longs.clear();
    for (uint32_t i = 0; i < src.n; ++i) {
        const uint64_t len = src.length(i);
        const Key k{static_cast<uint32_t>(len), i};
        if (len < threshold) shorts.push_back(k);
        else longs.push_back(k);
    }
    std::sort(shorts.begin(), shorts.end(), longer_first);
    std::sort(longs.begin(), longs.end(), longer_first);
}

template <class Fn>
void parallel_for(size_t n, Fn&& fn) {
    unsigned hw = std::thread::hardware_concurrency();
    const size_t workers = std::max<size_t>(1, std::min<size_t>(hw ? hw : 4, std::min<size_t>(n / 64 + 1, 32)));
    if (workers == 1) {
        for (size_t i = 0; i < n; ++i) fn(i);
        return;
    }
    std::atomic<size_t> next{0};
    std::vector<std::thread> pool;
    for (size_t w = 0; w < workers; ++w)
        pool.emplace_back([&] {
            for (;;) {
                const size_t begin = next.fetch_add(16);
                if (begin >= n) break;
                const size_t end = std::min(n, begin + 16);
                for (size_t i = begin; i < end; ++i) fn(i);
            }
        });
    for (auto& t : pool) t.join();
}

// The shard's sequences, longest first: every long sequence is at least as long as every short one, so the long
// pool followed by the short pool is sorted.
void local_pool(const SeqSource& src, uint64_t threshold, uint32_t shard_rank, uint32_t shard_count,
                std::vector<Key>& pool, uint32_t* n_short, uint32_t* n_long) {
    std::vector<Key> shorts_all, longs_all, shorts, longs;
    sorted_pools(src, threshold, shorts_all, longs_all);
    if (shard_count == 1) {
        shorts.swap(shorts_all);
        longs.swap(longs_all);
    } else {
        for (size_t p = 0; p < shorts_all.size(); ++p)
            if (snake(p, shard_count) == shard_rank) shorts.push_back(shorts_all[p]);
        for (size_t p = 0; p < longs_all.size(); ++p)
            if (shard_count - 1 - snake(p, shard_count) == shard_rank) longs.push_back(longs_all[p]);
    }
    *n_short = static_cast<uint32_t>(shorts.size());
    *n_long = static_cast<uint32_t>(longs.size());
    pool = std::move(longs);
    pool.insert(pool.end(), shorts.begin(), shorts.end());
}

// Groups of 64 over the sorted pool; rows padded to the group's longest member (its first) rounded up to 8.
// Returns the total number of chunks.
uint64_t build_groups(const std::vector<Key>& pool, std::vector<GroupDesc>& groups, uint64_t* padded_rows,
                      uint32_t* max_length) {
    const size_t n_groups = (pool.size() + kGroupSeqs - 1) / kGroupSeqs;
    groups.resize(n_groups);
    uint64_t chunk_cursor = 0;
    *padded_rows = 0;
    *max_length = 0;
    for (size_t g = 0; g < n_groups; ++g) {
        const uint32_t longest = pool[g * kGroupSeqs].len;
        const uint32_t n_chunks = (longest + kRowsPerChunk - 1) / kRowsPerChunk;
        groups[g] = GroupDesc{chunk_cursor, n_chunks, static_cast<uint32_t>(g * kGroupSeqs)};
        chunk_cursor += n_chunks;
        *padded_rows += static_cast<uint64_t>(n_chunks) * kRowsPerChunk;
        *max_length = std::max(*max_length, longest);
    }
    return chunk_cursor;
}

}  // namespace

void group_table(const SeqSource& src, uint64_t threshold, uint32_t shard_rank, uint32_t shard_count,
                 std::vector<GroupDesc>& groups, uint64_t* padded_rows) {
    std::vector<Key> pool;
    uint32_t n_short = 0, n_long = 0, max_length = 0;
    local_pool(src, threshold, shard_rank, shard_count, pool, &n_short, &n_long);
    build_groups(pool, groups, padded_rows, &max_length);
}

void shard_assignment(const SeqSource& src, uint64_t threshold, uint32_t shard_count,
                      std::vector<uint32_t>& shard_of) {
    shard_of.assign(src.n, 0);
    if (shard_count <= 1) return;
    std::vector<Key> shorts, longs;
    sorted_pools(src, threshold, shorts, longs);
    for (size_t p = 0; p < shorts.size(); ++p) shard_of[shorts[p].idx] = snake(p, shard_count);
    // The long pool is dealt starting from the opposite end so that the shard that received the
    // longest short sequence does not also receive the longest long one.
    for (size_t p = 0; p < longs.size(); ++p)
        shard_of[longs[p].idx] = shard_count - 1 - snake(p, shard_count);
}

std::string pack_database(const SeqSource& src, uint64_t threshold, uint32_t shard_rank,
                          uint32_t shard_count, PackedDb& out, bool* bad_code) {
    if (bad_code) *bad_code = false;
    if (shard_count < 1 || shard_rank >= shard_count) return "shard_rank must be < shard_count";
    for (uint32_t i = 0; i < src.n; ++i) {
        if (src.length(i) > 0xFFFFFFF0ull) return "sequence longer than 2^32-16 residues";
        if (src.length(i) && !src.data(i)) return "null sequence pointer with non-zero length";
    }

    out = PackedDb{};
    out.n_total = src.n;
    out.shard_rank = shard_rank;
    out.shard_count = shard_count;
    out.length_threshold = threshold;

    std::vector<Key> pool;
    local_pool(src, threshold, shard_rank, shard_count, pool, &out.n_short, &out.n_long);
    out.n_local = out.n_short + out.n_long;

    const size_t n_groups = (pool.size() + kGroupSeqs - 1) / kGroupSeqs;
    out.slot_index.assign(n_groups * kGroupSeqs, kNoSequence);
    out.slot_len.assign(n_groups * kGroupSeqs, 0);

    // member(g, s): the sequence in slot s of group g, or nullptr
    auto member = [&](size_t g, uint32_t s) -> const Key* {
        const size_t pos = g * kGroupSeqs + s;
        return pos < pool.size() ? &pool[pos] : nullptr;
    };

    const uint64_t chunk_cursor = build_groups(pool, out.groups, &out.padded_rows, &out.max_length);
    out.total_chunks = chunk_cursor;
    out.codes.assign(static_cast<size_t>(chunk_cursor) * 32 * 16, kPadCode);

    std::atomic<bool> bad{false};
    std::atomic<uint64_t> residues{0};
    parallel_for(n_groups, [&](size_t g) {
        const GroupDesc& gd = out.groups[g];
        uint8_t* base = out.codes.data() + static_cast<size_t>(gd.chunk_base) * 32 * 16;
        uint64_t res = 0;
        for (uint32_t s = 0; s < kGroupSeqs; ++s) {
            const Key* k = member(g, s);
            if (!k) break;
            const size_t slot = g * kGroupSeqs + s;
            out.slot_index[slot] = k->idx;
            out.slot_len[slot] = k->len;
            res += k->len;
            const uint32_t lane = s & 31, half = s >> 5;
            const uint8_t* codes = src.data(k->idx);
            for (uint32_t r0 = 0; r0 < k->len; r0 += kRowsPerChunk) {
                const uint32_t cnt = std::min(kRowsPerChunk, k->len - r0);
                uint8_t* dst = base + (static_cast<size_t>(r0 / kRowsPerChunk) * 32 + lane) * 16 + half * 8;
                for (uint32_t r = 0; r < cnt; ++r) {
                    const uint8_t c = codes[r0 + r];
                    if (c >= kAlphabet) bad.store(true, std::memory_order_relaxed);
                    dst[r] = c;
                }
            }
        }
        residues.fetch_add(res, std::memory_order_relaxed);
    });
    out.residues = residues.load();

    if (bad.load()) {
        if (bad_code) *bad_code = true;
        return "residue code outside the 24-symbol alphabet";
    }
    return {};
}

}  // namespace swb
