// pack.hpp -- host-side database packing for the B200 scoring path.
//
// Replaces the reference's per-search routing (partition_database, scheduler.hpp:56-65) and its
// per-chunk pointer gather (scheduler.hpp:156-160) with a one-off layout the kernels can stream.
//
// All sequences of a shard are sorted by (length desc, db_index asc) and cut into groups of 64
// (one warp: 32 lanes x 2 sequences, the two int16 halves of a DPX word).  Lane l of a group owns
// sorted positions base+l (half A, low 16 bits) and base+32+l (half B, high 16 bits).  Rows are
// padded with kPadCode to the group's longest member rounded up to 8.  Residues are interleaved
// so that one warp load of 512 contiguous bytes fetches 8 rows for all 64 sequences:
//
//       codes[(chunk*32 + lane)*16 + half*8 + r]        chunk = row / 8,  r = row % 8
//
// Routing by SearchConfig::length_threshold (scheduler.hpp:24,59-62) survives as bookkeeping
// (n_short / n_long feed SearchStats) and in the sharding below; execution-wise every group goes
// through the same tile-wavefront kernel, which gives a group as many cooperating warps as it has
// query tiles -- long sequences automatically get intra-task parallelism.
//
// Sharding: the long and the short sorted lists are each dealt over the shards in "snake" order,
// so every shard gets the same length distribution and residue count to within one sequence.
#pragma once
#include <cstdint>
#include <string>
#include <vector>

namespace swb {

constexpr uint32_t kAlphabet = 24;       // scoring.hpp:25
constexpr uint8_t kPadCode = 24;         // extra profile row: substitution score 0 against everything
constexpr uint32_t kGroupSeqs = 64;      // sequences per interleaved group
constexpr uint32_t kRowsPerChunk = 8;    // residues of one sequence per 16-byte lane slot
constexpr uint32_t kNoSequence = 0xFFFFFFFFu;

struct GroupDesc {
    uint64_t chunk_base;  // index of the group's first chunk, in units of (32 lanes x 16 B)
    uint32_t n_chunks;    // padded rows / 8
    uint32_t first_slot;  // index of the group's first entry in slot_index / slot_len
};

struct PackedDb {
    uint32_t n_total = 0, n_local = 0, n_short = 0, n_long = 0;
    uint32_t shard_rank = 0, shard_count = 1;
    uint32_t max_length = 0;
    uint64_t residues = 0;         // real residues in this shard
    uint64_t padded_rows = 0;      // sum over groups of padded rows (x64 = stored residues)
    uint64_t total_chunks = 0;
    uint64_t length_threshold = 0;

    std::vector<GroupDesc> groups;      // descending padded rows
    std::vector<uint32_t> slot_index;   // [n_groups*64] slot -> db_index, kNoSequence for unused slots
    std::vector<uint32_t> slot_len;     // [n_groups*64]
    std::vector<uint8_t> codes;         // total_chunks * 32 * 16 bytes
};

// Source of sequences: either pointer-per-sequence or flat codes + offsets.
struct SeqSource {
    const uint8_t* const* ptrs = nullptr;
    const uint32_t* lens = nullptr;
    const uint8_t* flat = nullptr;
    const uint64_t* offsets = nullptr;
    uint32_t n = 0;
    uint64_t length(uint32_t i) const { return lens ? lens[i] : offsets[i + 1] - offsets[i]; }   // lens alone is enough for planning
    const uint8_t* data(uint32_t i) const { return ptrs ? ptrs[i] : flat + offsets[i]; }
};

// shard_of[i] for every sequence.  Deterministic; depends only on the lengths.
void shard_assignment(const SeqSource& src, uint64_t threshold, uint32_t shard_count,
                      std::vector<uint32_t>& shard_of);

// The shard's group table alone (what pack_database would build), from the lengths only: for planning and tests.
void group_table(const SeqSource& src, uint64_t threshold, uint32_t shard_rank, uint32_t shard_count,
                 std::vector<GroupDesc>& groups, uint64_t* padded_rows);

// Returns empty string on success, else an error message; *bad_code set when a residue >= 24 was seen.
std::string pack_database(const SeqSource& src, uint64_t threshold, uint32_t shard_rank,
                          uint32_t shard_count, PackedDb& out, bool* bad_code);

}  // namespace swb
