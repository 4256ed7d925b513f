// Device side of the walk engine: graph view, the built-in programs as
// templated device functors, the samplers, and the persistent step kernel.
//
// Installed with the library (include/walkforge_b200/device/): a translation
// unit of user code instantiates walk_kernel for its own program type through
// include/walkforge_b200/device_program.cuh.
//
// Reference map (paths under /root/reference/proj):
//   GraphView            include/walkforge/graph.hpp:17-107 (CSR) + packed vertex words
//   Program<K>           include/walkforge/algorithms.hpp:20-193 via the WalkProgram
//                        concept (program.hpp:49-93): weight / update / finished / max_weight
//   Custom<U>            the same concept for a user's program type U (device_program.cuh)
//   move<P,S,F>          StepDriver::step, engine.hpp:342-426 (Direct / Tables / Gathered)
//   walk_kernel          run_sequential / run_interleaved (engine.hpp:440-504,
//                        interleave.hpp:391-556): a lane per walker, a global
//                        atomic query cursor refilling lanes (the GPU analogue of
//                        admit/refill, interleave.hpp:436-456, 531-538).
#pragma once

#include <cstdint>
#include <type_traits>

#include "../../walkforge_b200.h"
#include "rng.cuh"

namespace wf {

constexpr uint32_t kDegBits = 24;
constexpr uint32_t kDegEscape = (1u << kDegBits) - 1;  // degree >= this: read offsets
#ifndef WF_BLOCK
#define WF_BLOCK 256
#endif
constexpr int kBlock = WF_BLOCK;  // walk kernel threads per block
constexpr unsigned kFull = 0xFFFFFFFFu;
#ifndef WF_COOP_DEGREE
#define WF_COOP_DEGREE 32
#endif
constexpr uint32_t kCoopDegree = WF_COOP_DEGREE;  // gathered flows: warp-cooperative gather from this degree
constexpr int kMaxIndexedLabels = 6;  // 32 B label record: u64 base + 6 u32 group ends

enum Flow : int { kDirect = 0, kTables = 1, kGathered = 2 };
enum WalkerTypeE : int { kUnbiased = 0, kStatic = 1, kDynamic = 2 };  // program.hpp:17
// kRetry: an O-REJ trial rejected; the walker stays and draws its next trial
// in the kernel's next iteration (the same draws in the same order).
enum MoveResult : int { kDead = 0, kMoved = 1, kFault = 2, kRetry = 3 };

struct GraphView {
    uint32_t V;
    uint64_t E;
    const uint64_t* __restrict__ offsets;  // V+1
    const uint32_t* __restrict__ nbr;      // E, sorted per vertex when `sorted`
    const float* __restrict__ weights;     // E or null
    const double* __restrict__ weights64;  // E or null: the reference's f64 weights when they
                                           // are not all float32-exact (weights then mirrors them)
    const uint8_t* __restrict__ labels;    // E or null
    const uint64_t* __restrict__ vword;    // V: base << 24 | min(deg, escape)
    int sorted;
    // MetaPath label index (label-partitioned CSR): per vertex 32 B
    // {u64 base, u32 end[6]} and the stably partitioned neighbour array.
    const uint4* __restrict__ lab_rec;
    const uint32_t* __restrict__ lab_nbr;
    uint32_t label_count;
    // adjacency search index (sorted graphs), a sector-wide B-tree over each
    // neighbour list: level l (stride s_l = 16 * 8^l) holds
    // sidx[l][sidx_base(base, v, log2 s_l) + k] = nbr[base + s_l k], k < ceil(deg/s_l),
    // in sector-aligned groups of 8 heads.
    const uint32_t* sidx[9];
    int sidx_levels;
    // edge hash set (Node2Vec's distance test): open addressing over 32 B
    // buckets of four u64 keys (src << 32 | dst), load factor <= 1/2
    const unsigned long long* ehash;
    uint64_t ehash_buckets;
    // edge pre-filter (Node2Vec): blocked Bloom filter of unordered vertex
    // pairs, one 32 B sector per pair with kFilterBits bits set; "absent" is
    // exact (no false negatives), "maybe" falls through to the exact test
    const uint4* efilter;
    uint64_t efilter_sectors;  // power of two
    // instrumented runs only: [trials, search probes, scanned edges] (the
    // S_alg access counts of SURVEY 8d), else null
    unsigned long long* stats;
};

// A user program's functor bytes travel in the launch parameters (constant
// bank): a custom program of up to this size costs no memory traffic.
constexpr int kUserProgramBytes = 256;

struct ProgParams {
    alignas(16) unsigned char user[kUserProgramBytes];  // Custom<U>: the U object
    uint64_t stop_thr;  // PPR: ceil(termination * 2^53)
    uint32_t length;    // DeepWalk / Node2Vec / Uniform target length
    int weighted;
    double inv_a, inv_b, first, bound;  // Node2Vec (algorithms.hpp:87-90)
    double lo_w, hi_w;                  // min/max(1, 1/b): lazy O-REJ thresholds
    const uint32_t* __restrict__ schema;  // MetaPath (device copy)
    uint32_t schema_len;
};

struct WalkLaunch {
    GraphView g;
    const uint64_t* __restrict__ sview;  // sampling vertex words (exhausted -> degree 0)
    const uint4* __restrict__ alias;     // {thr lo, thr hi, first_dst, second_dst} per edge
    const double* __restrict__ its;      // cumulative per edge
    const double* __restrict__ rej_pstar;  // per vertex
    ProgParams prog;
    int qmode;
    uint32_t qsource;
    const uint32_t* __restrict__ qsources;
    uint64_t qid_begin;
    const uint64_t* __restrict__ qid_map;  // optional: cursor position -> qid
    uint64_t n_rows;
    uint32_t static_blocks;  // kClaim-row blocks dealt to each warp before the cursor
    uint64_t dyn_base;       // = warps * static_blocks * kClaim: first cursor-claimed row
    uint64_t seed_mixed;
    uint32_t trial_cap;
    uint32_t stride;
    uint32_t* __restrict__ paths;
    uint32_t* __restrict__ lengths;
    uint8_t* __restrict__ status;
    uint32_t* __restrict__ visit_counts;
    unsigned long long* steps_out;
    unsigned long long* overflow_out;
    unsigned long long* cursor;
    int* error_word;
    double* scratch;  // gathered ALIAS: per-warp weights + park areas for hub steps
    uint64_t scratch_stride;  // doubles per warp area (>= max degree)
    int use_label_index;
    int staged;  // rows 32 B-aligned: sector-sized path stores (PathStage)
    int alias_wide;                   // alias buckets are 32 B (2 x uint4) with dst vertex words
    int alias_idx;                    // alias buckets carry edge positions {first, second} in
                                      // E_v instead of destinations (programs that read the edge)
    const uint4* __restrict__ adj;    // Direct flows: {dst, 0, word lo, word hi} per edge, or null
    // Direct flows on graphs whose (dst, degree, base) pack into 64 bits: one
    // u64 per edge, dst | deg << adj8_vbits | base << (adj8_vbits + adj8_dbits)
    const unsigned long long* __restrict__ adj8;
    uint32_t adj8_vbits, adj8_dbits;
    const uint4* __restrict__ mp_adj; // MetaPath: per partitioned edge {dst, 0, next-group word} or null
    // Host streaming (run_to_host; all null otherwise).  Rows are grouped in
    // tiles of 2^tile_shift and chunks of 2^chunk_tiles_shift tiles.  Finished
    // rows report to their tile's word (rows << 40 | vertices); the report
    // that completes a tile adds it to its chunk's word (tiles << 40 |
    // vertices), and the one that completes a chunk publishes the chunk's
    // vertex total + 1 to host-mapped chunk_flag[chunk].
    unsigned long long* tile_word;
    unsigned long long* chunk_word;
    unsigned long long* chunk_flag;
    uint32_t tile_shift;
    uint32_t chunk_tiles_shift;
    // FROM_LIST sources arriving while the kernel runs: src_ready counts the
    // resident 2^src_shift-row blocks of the source list (written by the copy
    // stream behind each block's copy); null = all resident at launch
    const unsigned int* src_ready;
    uint32_t src_shift;
    uint64_t src_row0;  // rows of the list before this launch's first row
};

struct Walker {
    uint64_t row;
    Rng rng;
    uint64_t cur_base;
    uint64_t prev_base;
    uint32_t cur, prev;
    uint32_t cur_deg, prev_deg;
    uint32_t len;  // vertices on the path so far (moves + 1)
    uint32_t trials;  // O-REJ: trials of the current move so far (the cap, sampler.hpp:27)
    // vertex word of the destination when the sampler's load carried it
    uint64_t nb_word;
    bool have_nb;
    // nb_word holds the current vertex's raw word, not yet unpacked into
    // cur_base / cur_deg: the next move unpacks it after taking its first
    // draw, so the RNG arithmetic overlaps the word's load instead of waiting
    // behind the unpack's escape branch
    bool pend;
    // gathered flows: the outcome of this step's warp-cooperative gather
    // (coop_step) for a hub vertex, consumed by move(); kCoopNone otherwise
    uint8_t coop;
    uint32_t coop_pick;
};

enum CoopState : uint8_t { kCoopNone = 0, kCoopPick = 1, kCoopDead = 2, kCoopFault = 3 };

// ---- graph helpers -------------------------------------------------------------

// Random gathers (vertex words, buckets, neighbour ids, label records): cached
// in L2 only (ld.global.cg).  L1 hit rates on these are ~2 %, and letting L1
// allocate them made it request 2.8x the sectors the walk needs (ncu,
// profiles/).  Search probes keep __ldg: their last probes share a line.
#ifndef WF_LDR
#define WF_LDR "ld.global.cg"
#endif
__device__ __forceinline__ uint32_t ldr(const uint32_t* p) {
    uint32_t v;
    asm(WF_LDR ".u32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ uint64_t ldr(const uint64_t* p) {
    uint64_t v;
    asm(WF_LDR ".u64 %0, [%1];" : "=l"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ float ldr(const float* p) {
    float v;
    asm(WF_LDR ".f32 %0, [%1];" : "=f"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ uint4 ldr(const uint4* p) {
    uint4 v;
    asm(WF_LDR ".v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
    return v;
}
// One 256-bit load (sm_100: LDG.E.256): a whole 32 B sector in one request.
// Two 16 B loads of the same sector cost 2x the L2 lookups and made the L2
// fetch ~4 DRAM sectors per move (ncu, profiles/).
__device__ __forceinline__ void ldr256(const uint4* p, uint4& a, uint4& b) {
    asm(WF_LDR ".v8.u32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
        : "=r"(a.x), "=r"(a.y), "=r"(a.z), "=r"(a.w), "=r"(b.x), "=r"(b.y), "=r"(b.z), "=r"(b.w)
        : "l"(p));
}
// A random 16 B entry read as its aligned 32 B sector with one 256-bit load:
// measured (tools/randbw.cu) random 16 B requests sustain 20.9 G/s while 4 B,
// 8 B and 256-bit requests sustain 36.6 G/s — every random miss costs a 128 B
// line either way, so the wider load is free.
__device__ __forceinline__ uint4 ldr16(const uint4* p) {
    const uintptr_t a = reinterpret_cast<uintptr_t>(p);
    uint4 lo, hi;
    ldr256(reinterpret_cast<const uint4*>(a & ~static_cast<uintptr_t>(31)), lo, hi);
    return (a & 16) ? hi : lo;
}

// The one random request of a DeepWalk / MetaPath move (wide alias bucket,
// successor-decorated edge), with the .L2::64B prefetch-size qualifier: a
// miss then fetches 64 B from DRAM instead of the default 128 B line
// (tools/randbw_matrix.cu, profiles/r02_randbw_matrix.json: 2 vs 4 DRAM
// sectors per request).  C5 42.2 -> 43.0 G steps/s, C4 37.0 -> 37.4; the
// Node2Vec loads keep the default (its L2-resident filter and hash probes
// measured 4 % slower with it).
#ifndef WF_LDR_MOVE
#define WF_LDR_MOVE "ld.global.cg.L2::64B"
#endif
__device__ __forceinline__ void ldr256_move(const uint4* p, uint4& a, uint4& b) {
#ifdef WF_MOVE_EVICT_FIRST
    // experiment: evict-first L2 policy on the move's random line (keeps L2 for
    // the path rows' partial lines)
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    asm("ld.global.L2::cache_hint.L2::64B.v8.u32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8], %9;"
        : "=r"(a.x), "=r"(a.y), "=r"(a.z), "=r"(a.w), "=r"(b.x), "=r"(b.y), "=r"(b.z), "=r"(b.w)
        : "l"(p), "l"(pol));
#else
    asm(WF_LDR_MOVE ".v8.u32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
        : "=r"(a.x), "=r"(a.y), "=r"(a.z), "=r"(a.w), "=r"(b.x), "=r"(b.y), "=r"(b.z), "=r"(b.w)
        : "l"(p));
#endif
}
__device__ __forceinline__ uint4 ldr16_move(const uint4* p) {
    const uintptr_t a = reinterpret_cast<uintptr_t>(p);
    uint4 lo, hi;
    ldr256_move(reinterpret_cast<const uint4*>(a & ~static_cast<uintptr_t>(31)), lo, hi);
    return (a & 16) ? hi : lo;
}

// The O-REJ trial's random adjacency entry, marked evict-first in L2 (and a
// 64 B fetch): Node2Vec's pair filter (64 MiB, read at random by half the
// trials) then keeps more of its lines against the 2 GB adjacency stream —
// C3 6.55 -> 6.19 ms.  (Alone, without the policy, the 64 B fetch measured
// slower; the policy on DeepWalk's bucket loads slowed C5, whose only other
// L2 traffic is the path rows.)
__device__ __forceinline__ uint4 ldr16_stream(const uint4* p) {
    const uintptr_t a = reinterpret_cast<uintptr_t>(p);
    uint4 lo, hi;
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    asm("ld.global.L2::cache_hint.L2::64B.v8.u32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8], %9;"
        : "=r"(lo.x), "=r"(lo.y), "=r"(lo.z), "=r"(lo.w), "=r"(hi.x), "=r"(hi.y), "=r"(hi.z), "=r"(hi.w)
        : "l"(a & ~static_cast<uintptr_t>(31)), "l"(pol));
    return (a & 16) ? hi : lo;
}

// An edge's weight as the reference holds it (double, graph.hpp:102).
__device__ __forceinline__ double edge_weight(const GraphView& g, uint64_t e) {
    return g.weights64 ? __ldg(g.weights64 + e) : static_cast<double>(ldr(g.weights + e));
}

// A packed 8 B adjacency entry: the destination and its vertex word
// (base << kDegBits | deg) for the next move.
__device__ __forceinline__ uint32_t adj8_unpack(uint64_t e, uint32_t vbits, uint32_t dbits, uint64_t& word) {
    const uint32_t dst = static_cast<uint32_t>(e & ((1ull << vbits) - 1));
    const uint64_t deg = (e >> vbits) & ((1ull << dbits) - 1);
    word = ((e >> (vbits + dbits)) << kDegBits) | deg;
    return dst;
}

__device__ __forceinline__ void unpack_word(const GraphView& g, uint64_t w, uint32_t v,
                                            uint64_t& base, uint32_t& deg) {
    base = w >> kDegBits;
    deg = static_cast<uint32_t>(w & kDegEscape);
    if (deg == kDegEscape) {  // rare: very high degree
        base = ldr(g.offsets + v);
        deg = static_cast<uint32_t>(ldr(g.offsets + v + 1) - base);
    }
}

__device__ __forceinline__ void decode_vertex(const GraphView& g, const uint64_t* vw, uint32_t v,
                                              uint64_t& base, uint32_t& deg) {
    uint64_t w = ldr(vw + v);  // (L1-allocating ld.ca / ld.nc measured no different, C2)
    base = w >> kDegBits;
    deg = static_cast<uint32_t>(w & kDegEscape);
    if (deg == kDegEscape) {  // rare: very high degree
        base = ldr(g.offsets + v);
        deg = static_cast<uint32_t>(ldr(g.offsets + v + 1) - base);
    }
}

// Graph::has_edge (graph.cpp:182-188): std::binary_search on sorted lists,
// linear scan otherwise.  Membership only, so any exact search is equivalent.
__device__ __forceinline__ bool has_edge(const GraphView& g, uint64_t base, uint32_t deg,
                                         uint32_t dst, unsigned long long* probes = nullptr) {
    const uint32_t* ns = g.nbr + base;
    uint32_t np = 0;
    bool found = false;
    if (g.sorted) {
        uint32_t lo = 0, hi = deg;
        while (lo < hi) {
            uint32_t mid = (lo + hi) >> 1;
            ++np;
            if (__ldg(ns + mid) < dst) lo = mid + 1; else hi = mid;
        }
        found = lo < deg && (++np, __ldg(ns + lo) == dst);
    } else {
        for (uint32_t i = 0; i < deg && !found; ++i, ++np) found = __ldg(ns + i) == dst;
    }
    if (probes) atomicAdd(probes, static_cast<unsigned long long>(np));
    return found;
}

constexpr uint32_t kSidxBlock = 16;

constexpr int kSidxMaxLevels = 9;  // strides 2^4 .. 2^28: top level <= 8 heads for deg < 2^31

__host__ __device__ __forceinline__ int sidx_shift(int l) { return 4 + 3 * l; }

// Start of v's heads at a level with stride 2^sh: v owns ceil(deg / 2^sh) <=
// floor((base+deg) / 2^sh) - floor(base / 2^sh) + 1 words, so consecutive
// vertices never overlap and each level stays ~E/2^sh + V words (the
// sector-aligned variant padded every vertex to 8 words and fell out of L2:
// 10.2 vs 12.2 G steps/s on C3).
__host__ __device__ __forceinline__ uint64_t sidx_base(uint64_t base, uint64_t v, int sh) {
    return (base >> sh) + v;
}

// Membership of dst in the sorted adjacency of v (base, deg) through the
// sector B-tree: from the top level down, each level reads the <= 8 heads of
// the current group (two sectors, one round trip) and picks the last head
// <= dst; the chosen 16-id block is then read as 32 B sectors and compared in
// registers.  Same answer as std::binary_search (graph.cpp:182-188) in
// ~log8(deg/16) + 1 dependent rounds instead of ~log2(deg).
__device__ __forceinline__ bool has_edge_indexed(const GraphView& g, uint64_t base, uint32_t deg,
                                                 uint32_t v, uint32_t dst, unsigned long long* probes) {
    if (deg <= kSidxBlock || g.sidx_levels == 0) return has_edge(g, base, deg, dst, probes);
    int l = 0;
    while (((static_cast<uint64_t>(deg) + (1ull << sidx_shift(l)) - 1) >> sidx_shift(l)) > 8) {
        if (++l >= g.sidx_levels) return has_edge(g, base, deg, dst, probes);
    }
    uint32_t np = 0;
    uint64_t group = 0;  // first head index of the current group at level l
    uint64_t k = 0;
    for (; l >= 0; --l) {
        const int sh = sidx_shift(l);
        const uint64_t n = (static_cast<uint64_t>(deg) + (1ull << sh) - 1) >> sh;
        const uint32_t cnt = static_cast<uint32_t>((n - group) < 8 ? (n - group) : 8);
        // the group's <= 8 heads span at most two sectors of the compact level
        const uint64_t i0 = sidx_base(base, v, sh) + group;
        const uint32_t off = static_cast<uint32_t>(i0 & 7);
        const uint4* p = reinterpret_cast<const uint4*>(g.sidx[l] + (i0 & ~7ull));
        uint32_t c = 0;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            if (h == 1 && off + cnt <= 8) break;
            uint4 x, y;
            asm("ld.global.nc.v8.u32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                : "=r"(x.x), "=r"(x.y), "=r"(x.z), "=r"(x.w), "=r"(y.x), "=r"(y.y), "=r"(y.z), "=r"(y.w)
                : "l"(p + 2 * h));
            ++np;
            const uint32_t w[8] = {x.x, x.y, x.z, x.w, y.x, y.y, y.z, y.w};
#pragma unroll
            for (uint32_t j = 0; j < 8; ++j) {
                const uint32_t idx = 8 * h + j;
                c += (idx >= off && idx < off + cnt && w[j] <= dst) ? 1u : 0u;
            }
        }
        if (c == 0) {  // only at the top: dst below the smallest neighbour
            if (probes) atomicAdd(probes, static_cast<unsigned long long>(np));
            return false;
        }
        k = group + c - 1;
        group = k * 8;
    }
    // block k: neighbours [b0, b1)
    const uint64_t b0 = base + k * kSidxBlock;
    const uint64_t b1 = min(b0 + kSidxBlock, base + deg);
    bool found = false;
#pragma unroll
    for (int t = 0; t < 3; ++t) {
        const uint64_t s = (b0 & ~7ull) + 8ull * t;
        if (s < b1) {
            uint4 x, y;
            ldr256(reinterpret_cast<const uint4*>(g.nbr + s), x, y);
            ++np;
            uint32_t e[8] = {x.x, x.y, x.z, x.w, y.x, y.y, y.z, y.w};
#pragma unroll
            for (int i = 0; i < 8; ++i) found |= (s + i >= b0 && s + i < b1 && e[i] == dst);
        }
    }
    if (probes) atomicAdd(probes, static_cast<unsigned long long>(np));
    return found;
}

constexpr unsigned long long kHashEmpty = ~0ull;  // (2^32-1, 2^32-1) is never an edge

__host__ __device__ __forceinline__ uint64_t ehash_bucket(uint64_t key, uint64_t nb) {
    const uint64_t h = splitmix_mix(key ^ 0x6A09E667F3BCC909ULL);
#ifdef __CUDA_ARCH__
    return __umul64hi(h, nb);
#else
    return static_cast<uint64_t>((static_cast<unsigned __int128>(h) * nb) >> 64);
#endif
}

constexpr int kFilterBits = 4;  // bits per pair in its 256-bit sector

// The pair's sector and its kFilterBits bit positions (8 bits each) from one
// 64-bit mix of the unordered pair.
__host__ __device__ __forceinline__ uint64_t efilter_hash(uint32_t u, uint32_t v) {
    const uint32_t a = u < v ? u : v, b = u < v ? v : u;
    return splitmix_mix(((static_cast<uint64_t>(a) << 32) | b) ^ 0xBB67AE8584CAA73BULL);
}

// false: no edge between u and v in either direction (exact); true: maybe.
__device__ __forceinline__ bool efilter_maybe(const GraphView& g, uint32_t u, uint32_t v) {
    const uint64_t h = efilter_hash(u, v);
    uint4 lo, hi;
    ldr256(g.efilter + 2 * (h & (g.efilter_sectors - 1)), lo, hi);
    const uint32_t w[8] = {lo.x, lo.y, lo.z, lo.w, hi.x, hi.y, hi.z, hi.w};
    bool maybe = true;
#pragma unroll
    for (int i = 0; i < kFilterBits; ++i) {
        const uint32_t bit = static_cast<uint32_t>(h >> (32 + 8 * i)) & 255u;
        uint32_t word = 0;
#pragma unroll
        for (int k = 0; k < 8; ++k) word = (bit >> 5) == static_cast<uint32_t>(k) ? w[k] : word;
        maybe = maybe && ((word >> (bit & 31)) & 1u);
    }
    return maybe;
}

// Graph::has_edge (graph.cpp:182-188) as an exact hash-set lookup: one 32 B
// bucket (a single 256-bit load) answers almost every query — a random
// sector instead of a binary search's chain of dependent probes.  Same
// membership answer for sorted and unsorted adjacency alike.
__device__ __forceinline__ bool has_edge_hashed(const GraphView& g, uint32_t u, uint32_t v,
                                                unsigned long long* probes) {
    const unsigned long long key = (static_cast<unsigned long long>(u) << 32) | v;
    uint64_t b = ehash_bucket(key, g.ehash_buckets);
    uint32_t np = 0;
    bool found = false;
    for (;;) {
        uint4 x, y;
        ldr256(reinterpret_cast<const uint4*>(g.ehash + 4 * b), x, y);
        ++np;
        const unsigned long long k0 = (static_cast<unsigned long long>(x.y) << 32) | x.x;
        const unsigned long long k1 = (static_cast<unsigned long long>(x.w) << 32) | x.z;
        const unsigned long long k2 = (static_cast<unsigned long long>(y.y) << 32) | y.x;
        const unsigned long long k3 = (static_cast<unsigned long long>(y.w) << 32) | y.z;
        if (k0 == key || k1 == key || k2 == key || k3 == key) { found = true; break; }
        if (k0 == kHashEmpty || k1 == kHashEmpty || k2 == kHashEmpty || k3 == kHashEmpty) break;
        b = b + 1 == g.ehash_buckets ? 0 : b + 1;
    }
    if (probes) atomicAdd(probes, static_cast<unsigned long long>(np));
    return found;
}

// Node2Vec's "is dst a neighbour of prev" (algorithms.hpp:116-118).
__device__ __forceinline__ bool prev_has_edge(const GraphView& g, uint32_t prev, uint64_t prev_base,
                                              uint32_t prev_deg, uint32_t dst, unsigned long long* probes) {
    if (g.efilter) {
        if (probes) atomicAdd(probes, 1ull);  // the filter's sector is a request too
        if (!efilter_maybe(g, prev, dst)) return false;
    }
    if (g.ehash) return has_edge_hashed(g, prev, dst, probes);
    return has_edge_indexed(g, prev_base, prev_deg, prev, dst, probes);
}

// cumulative_upper_index, sampler.hpp:48-60.
__device__ __forceinline__ uint32_t upper_index(const double* cum, uint32_t n, double x) {
    uint32_t lo = 0, hi = n;
    while (lo < hi) {
        uint32_t mid = lo + (hi - lo) / 2;
        if (x < __ldg(cum + mid)) hi = mid; else lo = mid + 1;
    }
    return lo;
}

// ---- programs: the WalkProgram concept as device functors ------------------------
// Every program type P the kernel runs provides (all static, all inlined):
//   kind           WF_PROGRAM_* of a built-in, kCustomProgram for a user type
//   type           kUnbiased / kStatic / kDynamic (walker_type(), program.hpp:17)
//   prechecked     has finished() (PreCheckedProgram, program.hpp:81-84)
//   needs_edge     update() reads the traversed edge (the kernel then tracks its index)
//   checks_weights weight() results go through check_program_weight (engine.hpp:97-101)
//   weight(L, q, e)           q-dependent weight (gathered / O-REJ flows)
//   weight_static(L, src, e)  weight(nullptr, e) in static contexts (program.hpp:39-42)
//   update(L, q, e)           after each move, path already extended; true = finished
//   finished(L, q)            before the first move
// The built-ins read their constructor arguments from L.prog; a user's program
// (Custom<U> below) lives in L.prog.user.

constexpr int kCustomProgram = -1;

// Version of the launch record's meaning (WalkLaunch fields, scratch layout,
// program adapter): a user program library compiled against another value is
// refused at wf_session_create_custom (its kernels would misread the launch).
constexpr uint32_t kEngineAbi = 5;

template <int K>
struct Program;

template <>
struct Program<WF_PROGRAM_PPR> {  // algorithms.hpp:20-37
    static constexpr int kind = WF_PROGRAM_PPR;
    static constexpr int type = kUnbiased;
    static constexpr bool prechecked = false;
    static constexpr bool has_max_weight = true;
    static constexpr bool needs_edge = false;
    static constexpr bool checks_weights = false;
    __device__ static double weight(const WalkLaunch&, const Walker&, uint64_t) { return 1.0; }
    __device__ static double weight_static(const WalkLaunch&, uint32_t, uint64_t) { return 1.0; }
    // update draws the stop coin: uniform_real(1.0) < stop (algorithms.hpp:31)
    __device__ static bool update(const WalkLaunch& L, Walker& q, uint64_t) {
        return q.rng.bits53() < L.prog.stop_thr;
    }
    __device__ static bool finished(const WalkLaunch&, const Walker&) { return false; }
};

template <>
struct Program<WF_PROGRAM_UNIFORM> {  // algorithms.hpp:177-193
    static constexpr int kind = WF_PROGRAM_UNIFORM;
    static constexpr int type = kUnbiased;
    static constexpr bool prechecked = true;
    static constexpr bool has_max_weight = true;
    static constexpr bool needs_edge = false;
    static constexpr bool checks_weights = false;
    __device__ static double weight(const WalkLaunch&, const Walker&, uint64_t) { return 1.0; }
    __device__ static double weight_static(const WalkLaunch&, uint32_t, uint64_t) { return 1.0; }
    __device__ static bool update(const WalkLaunch& L, Walker& q, uint64_t) { return q.len >= L.prog.length; }
    __device__ static bool finished(const WalkLaunch& L, const Walker& q) { return q.len >= L.prog.length; }
};

template <>
struct Program<WF_PROGRAM_DEEPWALK> {  // algorithms.hpp:41-67
    static constexpr int kind = WF_PROGRAM_DEEPWALK;
    static constexpr int type = kStatic;
    static constexpr bool prechecked = true;
    static constexpr bool has_max_weight = true;
    static constexpr bool needs_edge = false;
    static constexpr bool checks_weights = false;
    __device__ static double weight_static(const WalkLaunch& L, uint32_t, uint64_t e) {
        return L.prog.weighted ? edge_weight(L.g, e) : 1.0;
    }
    __device__ static double weight(const WalkLaunch& L, const Walker&, uint64_t e) {
        return weight_static(L, 0, e);
    }
    __device__ static bool update(const WalkLaunch& L, Walker& q, uint64_t) { return q.len >= L.prog.length; }
    __device__ static bool finished(const WalkLaunch& L, const Walker& q) { return q.len >= L.prog.length; }
};

template <>
struct Program<WF_PROGRAM_NODE2VEC> {  // algorithms.hpp:79-133
    static constexpr int kind = WF_PROGRAM_NODE2VEC;
    static constexpr int type = kDynamic;
    static constexpr bool prechecked = true;
    static constexpr bool has_max_weight = true;
    static constexpr bool needs_edge = false;
    static constexpr bool checks_weights = false;
    __device__ static double weight(const WalkLaunch& L, const Walker& q, uint64_t e) {  // algorithms.hpp:103-119
        const ProgParams& p = L.prog;
        double w;
        if (q.len == 1) {
            w = p.first;
        } else {
            uint32_t dst = ldr(L.g.nbr + e);
            if (dst == q.prev) w = p.inv_a;
            else if (prev_has_edge(L.g, q.prev, q.prev_base, q.prev_deg, dst, L.g.stats ? L.g.stats + 1 : nullptr)) w = 1.0;
            else w = p.inv_b;
        }
        return p.weighted ? __dmul_rn(w, edge_weight(L.g, e)) : w;
    }
    __device__ static double weight_static(const WalkLaunch&, uint32_t, uint64_t) {
        return 0.0;  // never called: dynamic programs have no static tables
    }
    __device__ static bool update(const WalkLaunch& L, Walker& q, uint64_t) { return q.len >= L.prog.length; }
    __device__ static bool finished(const WalkLaunch& L, const Walker& q) { return q.len >= L.prog.length; }
};

template <>
struct Program<WF_PROGRAM_METAPATH> {  // algorithms.hpp:141-173
    static constexpr int kind = WF_PROGRAM_METAPATH;
    static constexpr int type = kDynamic;
    static constexpr bool prechecked = true;
    static constexpr bool has_max_weight = false;
    static constexpr bool needs_edge = false;
    static constexpr bool checks_weights = false;
    __device__ static double weight(const WalkLaunch& L, const Walker& q, uint64_t e) {  // algorithms.hpp:164-166
        return static_cast<uint32_t>(__ldg(L.g.labels + e)) == __ldg(L.prog.schema + (q.len - 1)) ? 1.0 : 0.0;
    }
    __device__ static double weight_static(const WalkLaunch&, uint32_t, uint64_t) { return 0.0; }
    __device__ static bool update(const WalkLaunch& L, Walker& q, uint64_t) { return q.len - 1 >= L.prog.schema_len; }
    __device__ static bool finished(const WalkLaunch& L, const Walker& q) { return q.len - 1 >= L.prog.schema_len; }
};

// ---- user programs ---------------------------------------------------------------
// The device face of the reference's Walker / EdgeRef (walker.hpp:24-45) that a
// user's program sees.  The walker's history is its current and previous
// vertex and its length (what the reference's own programs read: cur(),
// prev(), path.size(), moves()); the rest of the path is already in the
// output row.  The RNG is the walker's own stream; update() is the only place
// a program may draw from it (program.hpp:46-48).
class WalkerRng {
public:
    __device__ explicit WalkerRng(Rng& r) : r_(r) {}
    __device__ uint64_t next_u64() { return r_.next(); }                // rng.hpp:26-30
    __device__ uint32_t uniform_index(uint32_t n) { return r_.index(n); }  // rng.hpp:34-38
    __device__ double uniform_real(double bound) { return r_.real(bound); }  // rng.hpp:42-47

private:
    Rng& r_;
};

class WalkerView {
public:
    __device__ WalkerView(uint64_t id, uint32_t cur, uint32_t prev, uint32_t len, Rng* rng)
        : id_(id), cur_(cur), prev_(prev), len_(len), rng_(rng) {}
    __device__ uint64_t id() const { return id_; }
    __device__ uint32_t cur() const { return cur_; }
    __device__ uint32_t prev() const { return prev_; }  // valid after one move
    __device__ uint64_t path_size() const { return len_; }
    __device__ uint64_t moves() const { return len_ - 1; }
    // Only in update(): weight() must not draw (program.hpp:46-48).
    __device__ WalkerRng rng() const { return WalkerRng(*rng_); }

private:
    uint64_t id_;
    uint32_t cur_, prev_, len_;
    Rng* rng_;
};

class EdgeRef {  // walker.hpp:37-45: lazy, a program touches only what it reads
public:
    __device__ EdgeRef(const GraphView& g, uint32_t src, uint64_t index) : g_(g), src_(src), index_(index) {}
    __device__ uint32_t src() const { return src_; }
    __device__ uint64_t index() const { return index_; }
    __device__ uint32_t dst() const { return ldr(g_.nbr + index_); }
    __device__ double weight() const { return edge_weight(g_, index_); }
    __device__ uint32_t label() const { return __ldg(g_.labels + index_); }

private:
    const GraphView& g_;
    uint32_t src_;
    uint64_t index_;
};

__device__ __forceinline__ uint64_t walker_qid(const WalkLaunch& L, const Walker& q) {
    return L.qid_map ? __ldg(L.qid_map + q.row) : L.qid_begin + q.row;
}

// The walk engine's view of a user program type U (device_program.cuh).  U is
// trivially copyable, fits kUserProgramBytes, and declares
//   static constexpr wf_walker_type walker_type = ...;
//   __device__ double weight(const WalkerView* q, const EdgeRef& e) const;  // q null: static
//   __device__ bool update(WalkerView& q, const EdgeRef& e) const;
// and optionally max_weight() (host + device), finished(const WalkerView&).
template <class U, class = void>
struct has_finished : std::false_type {};
template <class U>
struct has_finished<U, std::void_t<decltype(std::declval<const U&>().finished(std::declval<const WalkerView&>()))>>
    : std::true_type {};
template <class U, class = void>
struct has_max_weight_fn : std::false_type {};
template <class U>
struct has_max_weight_fn<U, std::void_t<decltype(std::declval<const U&>().max_weight())>> : std::true_type {};

template <class U>
struct Custom {
    static_assert(std::is_trivially_copyable<U>::value, "a device program must be trivially copyable");
    static_assert(sizeof(U) <= kUserProgramBytes, "a device program must fit kUserProgramBytes");
    static constexpr int kind = kCustomProgram;
    static constexpr int type = static_cast<int>(U::walker_type);
    static constexpr bool prechecked = has_finished<U>::value;
    static constexpr bool has_max_weight = has_max_weight_fn<U>::value;
    static constexpr bool needs_edge = true;
    static constexpr bool checks_weights = true;
    __device__ static const U& self(const WalkLaunch& L) { return *reinterpret_cast<const U*>(L.prog.user); }
    __device__ static WalkerView view(const WalkLaunch& L, const Walker& q) {
        return WalkerView(walker_qid(L, q), q.cur, q.prev, q.len, const_cast<Rng*>(&q.rng));
    }
    __device__ static double weight(const WalkLaunch& L, const Walker& q, uint64_t e) {
        const WalkerView v = view(L, q);
        return self(L).weight(&v, EdgeRef(L.g, q.cur, e));
    }
    __device__ static double weight_static(const WalkLaunch& L, uint32_t src, uint64_t e) {
        return self(L).weight(static_cast<const WalkerView*>(nullptr), EdgeRef(L.g, src, e));
    }
    __device__ static bool update(const WalkLaunch& L, Walker& q, uint64_t e) {
        WalkerView v = view(L, q);
        return self(L).update(v, EdgeRef(L.g, q.prev, e));  // EdgeRef{&g, walker.prev(), edge}, engine.hpp:481
    }
    __device__ static bool finished(const WalkLaunch& L, const Walker& q) {
        if constexpr (has_finished<U>::value) return self(L).finished(view(L, q));
        else return false;
    }
};

// ---- samplers ------------------------------------------------------------------

__device__ __forceinline__ void raise_device(const WalkLaunch& L, int code) {
    atomicCAS(L.error_word, 0, code);
}

// check_program_weight (engine.hpp:97-101) for programs whose weights are not
// known good: a negative or non-finite weight raises ContractError at the
// next sync; the walk stops as a fault.
template <class P>
__device__ __forceinline__ bool weight_ok(const WalkLaunch& L, double w) {
    if constexpr (P::checks_weights) {
        if (!(w >= 0.0 && w <= 1.7976931348623157e308)) {
            raise_device(L, WF_ERR_CONTRACT);
            return false;
        }
    }
    return true;
}

// O-REJ accept test (rej_generate, sampler.hpp:152-164 with the program weight
// evaluated lazily, engine.hpp:356-364).  Node2Vec evaluates only as much of
// its weight as y needs: every weight out of a vertex lies in {1/a, 1, 1/b}
// (times w_e when weighted) so y below / above the candidates decides without
// the adjacency search.  Same accept decisions, same draws — bit-exact.
// Returns 1 accept, 0 reject, -1 contract fault.
template <class P>
__device__ __forceinline__ int orej_accept(const WalkLaunch& L, const Walker& q, uint64_t e, double y,
                                           uint32_t dst) {
    if constexpr (P::kind == WF_PROGRAM_NODE2VEC) {
        const ProgParams& p = L.prog;
        double ew = p.weighted ? edge_weight(L.g, e) : 1.0;
        auto scaled = [&](double w) { return p.weighted ? __dmul_rn(w, ew) : w; };
        if (q.len == 1) return y < scaled(p.first);
        if (dst == q.prev) return y < scaled(p.inv_a);
        if (y < scaled(p.lo_w)) return 1;
        if (!(y < scaled(p.hi_w))) return 0;
        bool common = prev_has_edge(L.g, q.prev, q.prev_base, q.prev_deg, dst, L.g.stats ? L.g.stats + 1 : nullptr);
#ifdef WF_DIAG_COMMON
        if (common && L.g.stats) atomicAdd(L.g.stats + 2, 1ull);  // diagnostics: distance tests answered "edge"
#endif
        return y < scaled(common ? 1.0 : p.inv_b);
    } else {
        const double w = P::weight(L, q, e);
        if (!weight_ok<P>(L, w)) return -1;
        return y < w;
    }
}

// Vose's alias construction (sampler.hpp:89-120) for ONE bucket x, replayed
// without the FIFO worklists: the small queue is [initial smalls ascending] ++
// [larges in demotion order] and larges are demoted in ascending order, so
// ascending cursors (or bitmasks) over the scaled weights w_i * n / sum
// (sampler.hpp:97) reproduce it exactly; a demoted large's final value is
// kept until it is consumed as a small.  Returns the split of bucket x and
// its alias index (x itself when it is a leftover at probability 1).

// The replay for a light vertex (d < kCoopDegree <= 64) whose
// weights sit in a lane-local array: the scaled weights replace them in
// place, the worklists are bitmasks (initial smalls, larges not yet head,
// demoted larges — each consumed lowest index first, which is the FIFO order
// since larges are demoted in ascending order), and a demoted large's final
// value overwrites its own slot, so no scan ever re-reads a weight.
__device__ __forceinline__ void vose_bucket_local(uint32_t n, double sum, double* w, uint32_t x, double& split_out,
                                                  uint32_t& second_out) {
    static_assert(kCoopDegree <= 64, "bitmask worklists");
    uint64_t largem = 0;
    for (uint32_t i = 0; i < n; ++i) {
        w[i] = w[i] * n / sum;  // sampler.hpp:97
        if (w[i] >= 1.0) largem |= 1ull << i;
    }
    uint64_t sq = (n == 64 ? ~0ull : (1ull << n) - 1) & ~largem;  // initial smalls not yet popped
    uint64_t lq = largem;                                           // larges not yet head
    uint64_t dq = 0;                                                // demoted larges not yet popped
    if (lq) {
        uint32_t l = __ffsll(static_cast<long long>(lq)) - 1;
        lq &= lq - 1;
        double lval = w[l];
        for (;;) {  // sampler.hpp:103-111
            uint32_t s;
            if (sq) {
                s = __ffsll(static_cast<long long>(sq)) - 1;
                sq &= sq - 1;
            } else if (dq) {
                s = __ffsll(static_cast<long long>(dq)) - 1;
                dq &= dq - 1;
            } else {
                break;
            }
            const double sval = w[s];
            if (s == x) {
                split_out = sval;
                second_out = l;
                return;
            }
            lval -= 1.0 - sval;
            if (lval < 1.0) {
                w[l] = lval;
                dq |= 1ull << l;
                if (!lq) break;
                l = __ffsll(static_cast<long long>(lq)) - 1;
                lq &= lq - 1;
                lval = w[l];
            }
        }
    }
    split_out = 1.0;  // leftover: probability exactly 1, no alias (sampler.hpp:112-119)
    second_out = x;
}

// ---- Vose's worklists for a hub, by a warp ---------------------------------------
// The replay for bucket x over a hub's weights (`row`, n
// entries, summed to `total`), with the serial chain on one lane.  Vose's
// pairing loop is an order-dependent fp64 chain (lval -= 1 - sval), so it
// cannot be split; everything around it can.  The warp first turns the row
// into scaled weights (w * n / total, sampler.hpp:97, one division each) and
// compacts them: the smalls' values in index order to the front of `park`,
// the larges' values to its back (the j-th large at park[n-1-j]), the larges'
// indices over the row's front.  Lane 0 then runs the chain over 128-entry
// batches the warp stages in shared memory — for the smalls their deficits
// fl(1 - s), computed by the staging lanes (the same rounding as the chain's
// own subtraction), so a pairing is one subtraction and one compare — and
// writes each demoted large's final value over its own slot, where the
// second phase (demoted larges consumed as smalls, in demotion order) reads
// it.  `row` is overwritten.
constexpr uint32_t kVoseStage = 128;

__device__ __forceinline__ void vose_bucket_staged(uint32_t n, double* __restrict__ row, double total, uint32_t x,
                                                   double* __restrict__ park, double& split_out,
                                                   uint32_t& second_out) {
    __shared__ double vose_stage[kBlock / 32][2][kVoseStage + 2];
    const int lane = threadIdx.x & 31;
    double* tb = vose_stage[threadIdx.x >> 5][0];  // deficits: smalls (phase 1) / demoted larges (phase 2)
    double* lb = vose_stage[threadIdx.x >> 5][1];  // larges' initial values
    uint32_t* li = reinterpret_cast<uint32_t*>(row);
    const unsigned lt = (1u << lane) - 1;
    // 1. scaled weights, compacted; four 32-entry rounds per load batch
    uint32_t ns = 0, nl = 0, xinfo = 0;  // x: small << 31 | rank among its class
    for (uint32_t c0 = 0; c0 < n; c0 += 128) {
        double v[4];
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            const uint32_t i = c0 + 32 * r + lane;
            v[r] = i < n ? row[i] : 0.0;
        }
        __syncwarp();  // the batch is read before the large indices overwrite the row's front
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            const uint32_t i = c0 + 32 * r + lane;
            const double sc = v[r] * n / total;
            const bool valid = i < n, sm = valid && sc < 1.0;
            const unsigned bs = __ballot_sync(kFull, sm), bl = __ballot_sync(kFull, valid && !sm);
            const uint32_t rs = ns + __popc(bs & lt), rl = nl + __popc(bl & lt);
            if (sm) {
                park[rs] = sc;
            } else if (valid) {
                park[n - 1 - rl] = sc;
                li[rl] = i;
            }
            if (i == x) xinfo = sm ? (0x80000000u | rs) : rl;
            ns += __popc(bs);
            nl += __popc(bl);
        }
    }
    xinfo = __shfl_sync(kFull, xinfo, x & 31);
    const bool xs = xinfo >> 31;
    const uint32_t xr = xinfo & 0x7FFFFFFFu;
    __syncwarp();
    // 2. the chain (sampler.hpp:103-111), lane 0, batch by batch
    uint32_t k = 0, j = 0, dq = 0;  // next small, head large, next demoted large to consume
    uint32_t tbase = 0, tlen = 0, lbase = 0, llen = 0;
    int tphase = 0;                 // what tb holds: 0 nothing, 1 smalls, 2 demoted larges
    int phase = 1;
    bool head_pending = true, done = nl == 0, found = false;
    double lval = 0.0;
    while (!done) {
        // stage what lane 0 needs next (uniform decisions)
        if (phase == 1 && k < ns && !(tphase == 1 && k < tbase + tlen)) {
            tbase = k;
            tlen = min(kVoseStage, ns - k);
            for (uint32_t t = lane; t < tlen; t += 32) tb[t] = 1.0 - park[k + t];
            tphase = 1;
        } else if (phase == 2 && dq < j && !(tphase == 2 && dq < tbase + tlen)) {
            tbase = dq;
            tlen = min(kVoseStage, j - dq);
            for (uint32_t t = lane; t < tlen; t += 32) tb[t] = 1.0 - park[n - 1 - (dq + t)];
            tphase = 2;
        }
        if (j < nl && !(j >= lbase && j < lbase + llen)) {
            lbase = j;
            llen = min(kVoseStage, nl - j);
            for (uint32_t t = lane; t < llen; t += 32) lb[t] = park[n - 1 - (j + t)];
        }
        __syncwarp();
        if (lane == 0) {
            if (head_pending) {
                lval = lb[j - lbase];
                head_pending = false;
            }
            // pairings until x, the batch's end or the larges' batch end
            uint32_t& cur = phase == 1 ? k : dq;
            const uint32_t stop_x = (phase == 1) == xs ? xr : 0xFFFFFFFFu;
            const uint32_t stop = min(tbase + tlen, stop_x);
            const uint32_t lend = lbase + llen;  // <= nl
            // the next head's value is loaded ahead (off the chain's critical
            // path); the chain itself is one subtraction and one compare
            const double* tp = tb - tbase;
            const double* lp = lb - lbase;
            double* pj = park + (n - 1 - j);
            double nv = j + 1 < lend ? lp[j + 1] : 0.0;
            const uint32_t qcap = phase == 2 ? 0u : 0xFFFFFFFFu;  // phase 2: the queue may not pass j
            uint32_t c = cur, jj = j;
            bool out = false;
            // deficits two ahead in registers, unrolled by two so each stays
            // in its own register (tb has kVoseStage + 2 slots: the look-ahead
            // never leaves the stage); the next head's value is loaded ahead
            double ta = tp[c], tb2 = tp[c + 1];
            auto pair = [&](double& tr) -> bool {  // one pairing; true: leave the batch
                lval -= tr;
                tr = tp[c + 2];
                ++c;
                if (lval < 1.0) {
                    *pj-- = lval;  // the demoted value, read back in phase 2
                    ++jj;
                    if (jj >= lend || (c >= jj && qcap == 0u)) return out = true;
                    lval = nv;
                    nv = jj + 1 < lend ? lp[jj + 1] : 0.0;
                }
                return false;
            };
            for (;;) {
                if (c >= stop || pair(ta)) break;
                if (c >= stop || pair(tb2)) break;
            }
            cur = c;
            j = jj;
            if (j == nl) {
                done = true;  // no large left: every remaining bucket is a leftover
            } else if (!out && cur == stop_x) {
                done = found = true;  // x is paired with the head large
            } else if (j >= lend) {
                head_pending = true;
            } else if (phase == 2 && dq >= j) {
                done = true;  // nothing left to pair: x is a leftover
            }
            if (!done && phase == 1 && k >= ns) phase = 2;
            if (!done && phase == 2 && dq >= j) done = true;
        }
        k = __shfl_sync(kFull, k, 0);
        j = __shfl_sync(kFull, j, 0);
        dq = __shfl_sync(kFull, dq, 0);
        phase = __shfl_sync(kFull, phase, 0);
        done = __shfl_sync(kFull, done, 0);
        head_pending = __shfl_sync(kFull, head_pending, 0);
        __syncwarp();  // lane 0's demoted values are visible to the next batch's loads
    }
    found = __shfl_sync(kFull, found, 0);
    if (found) {  // bucket x: its own (final) value and the head large
        split_out = xs ? park[xr] : park[n - 1 - xr];
        second_out = li[j];
    } else {
        split_out = 1.0;  // leftover: probability exactly 1, no alias (sampler.hpp:112-119)
        second_out = x;
    }
}

// Index of the j-th (0-based) positive entry of row[0, n), by the warp: 256
// entries per load batch, batches skipped on their ballot counts.
__device__ __forceinline__ uint32_t warp_select_positive(const double* __restrict__ row, uint32_t n, uint64_t j) {
    const int lane = threadIdx.x & 31;
    uint64_t seen = 0;
    for (uint32_t c0 = 0; c0 < n; c0 += 256) {
        unsigned m[8];
        uint32_t tot = 0;
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            const uint32_t i = c0 + 32 * r + lane;
            m[r] = __ballot_sync(kFull, i < n && row[i] > 0.0);
            tot += __popc(m[r]);
        }
        if (seen + tot <= j) {
            seen += tot;
            continue;
        }
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            const uint32_t pc = __popc(m[r]);
            if (seen + pc > j) return c0 + 32 * r + __fns(m[r], 0, static_cast<int>(j - seen) + 1);
            seen += pc;
        }
    }
    return n;  // not reached: j < the number of positive entries
}

// The replay in closed form when every positive weight has the same value
// (MetaPath's 0/1 weights, unweighted programs).  Then every large starts at
// c = w * n / sum (sampler.hpp:97, the same expression) and every small is a
// zero, and the chain is exact arithmetic on multiples of ulp(c):
//   phase 1 — each large absorbs K = floor(c) zeros (lval -= 1 exactly) and
//     is demoted at f = c - K, so the zero of rank r pairs with the large of
//     rank r / K;
//   phase 2 — the D = Z / K larges demoted in phase 1 (Z zeros) are consumed
//     in rank order, each with deficit t = 1 - f: head D (at c - Z mod K)
//     takes a0 = floor((v0 - 1) / t) + 1 of them, every later head
//     ac = floor((c - 1) / t) + 1, and the larges those heads demote queue
//     behind them (position = rank), so the first D positions are consumed
//     by that formula alone.
// Returns false for the one case that needs the chain: x a large the first
// phase did not demote.  Checked against the reference's tables and walks.
__device__ __forceinline__ bool vose_bucket_uniform(uint32_t n, uint32_t m, double w, double total, uint32_t x,
                                                    bool xpos, uint32_t xrank, const double* __restrict__ row,
                                                    double& split_out, uint32_t& second_out) {
    const double c = w * n / total;
    if (m == n || !(c >= 1.0) || !(c < 4503599627370496.0)) {  // no smalls (c == 1): all leftovers
        if (m != n) return false;
        split_out = 1.0;
        second_out = x;
        return true;
    }
    const uint64_t K = static_cast<uint64_t>(c);
    const double f = c - static_cast<double>(K);  // exact
    const uint64_t Z = n - m;
    if (!xpos) {  // phase 1
        const uint64_t j = xrank / K;
        if (j < m) {
            split_out = 0.0;
            second_out = warp_select_positive(row, n, j);
        } else {
            split_out = 1.0;
            second_out = x;
        }
        return true;
    }
    const uint64_t D = Z / K;
    if (xrank >= D) return false;
    // phase 2 over the first-generation entries, in units of u = ulp(c)
    const int e = ilogb(c) - 52;
    const double t = 1.0 - f;
    const double v0 = c - static_cast<double>(Z - D * K);
    const uint64_t T = static_cast<uint64_t>(ldexp(t, -e));
    const uint64_t a0 = static_cast<uint64_t>(ldexp(v0 - 1.0, -e)) / T + 1;
    const uint64_t ac = static_cast<uint64_t>(ldexp(c - 1.0, -e)) / T + 1;
    const uint64_t head = xrank < a0 ? D : D + 1 + (xrank - a0) / ac;
    if (head < m) {
        split_out = f;
        second_out = warp_select_positive(row, n, head);
    } else {
        split_out = 1.0;
        second_out = x;
    }
    return true;
}

// Deferred unpack of the current vertex word (Walker::pend): on for every
// program but Node2Vec, whose O-REJ kernel measured 3 % slower with it.
template <class P>
constexpr bool kDeferWord = P::kind != WF_PROGRAM_NODE2VEC;

// One move: StepDriver::step (engine.hpp:342-426).  Draw order per sampler is
// the reference contract (engine.hpp:330-333): NAIVE x; ITS x_real; ALIAS x
// then y; REJ / O-REJ (x, y) per trial; dead ends consume no draws.  `edge`
// (the global index of the traversed edge) is produced only for programs
// whose update() reads it (P::needs_edge).
template <class P, int S, int F>
__device__ __forceinline__ int move(const WalkLaunch& L, Walker& q, uint32_t& dst, uint64_t& edge) {
    if constexpr (kDeferWord<P>) {
        if (q.pend) {
            unpack_word(L.g, q.nb_word, q.cur, q.cur_base, q.cur_deg);
            q.pend = false;
        }
    }
    const uint32_t d = q.cur_deg;
    const uint64_t base = q.cur_base;
    if (L.g.stats && P::kind == WF_PROGRAM_METAPATH) {
        // instrumented runs: the reference's gather scans every label of the
        // current vertex (ceil(d_v / 32) u8-label sectors per step)
        const uint64_t d_v = ldr(L.g.offsets + q.cur + 1) - ldr(L.g.offsets + q.cur);
        atomicAdd(L.g.stats + 4, static_cast<unsigned long long>((d_v + 31) / 32));
        atomicAdd(L.g.stats + 5, 1ull);
    }
    if (d == 0) return kDead;
    uint32_t pick = 0;
    if constexpr (F == kDirect) {
        if constexpr (S == WF_SAMPLER_NAIVE) {
            pick = q.rng.index(d);
        } else {  // O-REJ
            // One trial per call.  A rejected trial returns kRetry and the
            // kernel's next iteration draws the next one: in a warp, a lane
            // with a second trial (~6 % of Node2Vec moves, so most warp
            // iterations on C3) no longer holds the other 31 at the loop's
            // reconvergence point for a whole extra dependent chain.
            if (q.trials >= L.trial_cap) {
                raise_device(L, WF_ERR_REJECTION_CAP);
                return kFault;
            }
            ++q.trials;
            if (L.g.stats) atomicAdd(L.g.stats, 1ull);
            uint32_t x = q.rng.index(d);
            double y = q.rng.real(L.prog.bound);
            // one sector per trial: the candidate's id (and, with the
            // decorated adjacency, its vertex word for the next step)
            uint32_t dx;
            uint64_t wx = 0;
            if (L.adj8) {
                dx = adj8_unpack(ldr(reinterpret_cast<const uint64_t*>(L.adj8) + base + x), L.adj8_vbits,
                                 L.adj8_dbits, wx);
            } else if (L.adj) {
                uint4 a = ldr16_stream(L.adj + base + x);
                dx = a.x;
                wx = (static_cast<uint64_t>(a.w) << 32) | a.z;
            } else {
                dx = ldr(L.g.nbr + base + x);
            }
            if (L.g.stats && P::kind == WF_PROGRAM_NODE2VEC && q.len > 1 && dx != q.prev) {
                // instrumented runs: the reference's weight() binary-searches
                // adj(prev) on every such trial (ceil(log2(d_prev+1)) probes)
                atomicAdd(L.g.stats + 3, static_cast<unsigned long long>(32 - __clz(q.prev_deg)));
            }
            const int acc = orej_accept<P>(L, q, base + x, y, dx);
            if (acc < 0) return kFault;
            if (!acc) return kRetry;
            q.trials = 0;
            dst = dx;
            if constexpr (P::needs_edge) edge = base + x;
            if (L.adj || L.adj8) {
                q.nb_word = wx;
                q.have_nb = true;
            }
            return kMoved;
        }
    } else if constexpr (F == kTables) {
        if constexpr (S == WF_SAMPLER_ALIAS) {
            uint32_t x = q.rng.index(d);
            if (L.alias_wide) {
                // 32 B bucket = one sector: {thr, first_dst, second_dst} and the
                // destinations' own vertex words, so the next step needs no
                // dependent vertex-word load (one random sector per move).
                uint4 b, w;
                ldr256_move(L.alias + 2 * (base + x), b, w);
                uint64_t thr = (static_cast<uint64_t>(b.y) << 32) | b.x;
                bool first = q.rng.bits53() < thr;  // y < split <=> k < ceil(split 2^53)
                dst = first ? b.z : b.w;
                q.nb_word = first ? (static_cast<uint64_t>(w.y) << 32) | w.x
                                  : (static_cast<uint64_t>(w.w) << 32) | w.z;
                q.have_nb = true;
                return kMoved;
            }
            uint4 b = ldr16(L.alias + base + x);
            uint64_t thr = (static_cast<uint64_t>(b.y) << 32) | b.x;
            const bool first = q.rng.bits53() < thr;  // y < split <=> k < ceil(split 2^53)
            if (L.alias_idx) {
                // {thr, first, second} as positions in E_v (EngineAliasSlot's
                // first / second, engine.hpp:22-28): the edge, then its destination
                pick = first ? b.z : b.w;
            } else {
                dst = first ? b.z : b.w;
                return kMoved;
            }
        } else if constexpr (S == WF_SAMPLER_ITS) {
            const double* cum = L.its + base;
            double x = q.rng.real(__ldg(cum + d - 1));
            pick = upper_index(cum, d, x);
        } else {  // REJ with p* per vertex
            // one trial per call, like O-REJ (kRetry)
            if (q.trials >= L.trial_cap) {
                raise_device(L, WF_ERR_REJECTION_CAP);
                return kFault;
            }
            ++q.trials;
            if (L.g.stats) atomicAdd(L.g.stats, 1ull);
            const double ps = __ldg(L.rej_pstar + q.cur);
            uint32_t x = q.rng.index(d);
            double y = q.rng.real(ps);
            if (!(y < P::weight_static(L, q.cur, base + x))) return kRetry;
            q.trials = 0;
            pick = x;
        }
    } else {  // Gathered: gather (engine.hpp:134-184) without the scratch table
        if constexpr (P::kind == WF_PROGRAM_METAPATH && S == WF_SAMPLER_ITS) {
            if (L.use_label_index) {
                // label-partitioned CSR: q.cur_base / q.cur_deg already frame the
                // group of edges labelled schema[moves]; the reference picks the
                // j-th matching edge in CSR order with j = floor(uniform_real(m))
                // (cumulative table over 0/1 weights), which is the j-th edge of
                // the stably partitioned group.
                double x = q.rng.real(static_cast<double>(d));
                const uint32_t j = static_cast<uint32_t>(x);
                if (L.mp_adj) {
                    // {dst, -, group word of dst for the next schema label}: the
                    // next move's label group arrives with this one load
                    uint4 a = ldr16_move(L.mp_adj + base + j);
                    dst = a.x;
                    const uint64_t w = (static_cast<uint64_t>(a.w) << 32) | a.z;
                    if (w != ~0ull) {
                        q.nb_word = w;
                        q.have_nb = true;
                    }
                    return kMoved;
                }
                dst = ldr(L.g.lab_nbr + base + j);
                return kMoved;
            }
        }
        if (q.coop != kCoopNone) {  // the warp gathered this hub step (coop_step)
            const uint8_t c = q.coop;
            q.coop = kCoopNone;
            if (c == kCoopDead) return kDead;
            if (c == kCoopFault) return kFault;
            if constexpr (P::needs_edge) edge = base + q.coop_pick;
            dst = ldr(L.g.nbr + base + q.coop_pick);
            return kMoved;
        }
        double sum = 0.0, mx = 0.0;
        if (L.g.stats) atomicAdd(L.g.stats + 2, static_cast<unsigned long long>(d));
        // below kCoopDegree (hubs go through coop_step) the weights stay in a
        // lane-local array, so each is evaluated (for Node2Vec: an adjacency
        // test) once per step
        double wl[kCoopDegree];
        const bool local = d < kCoopDegree;
        for (uint32_t i = 0; i < d; ++i) {
            double w = P::weight(L, q, base + i);
            if (!weight_ok<P>(L, w)) return kFault;
            if (local) wl[i] = w;
            sum += w;
            mx = w > mx ? w : mx;
        }
        if (!(sum > 0.0)) return kDead;
        if constexpr (S == WF_SAMPLER_ITS) {
            double x = q.rng.real(sum);  // == cumulative[d-1]: same sequential sum
            double run = 0.0;
            pick = d - 1;
            for (uint32_t i = 0; i < d; ++i) {
                run += local ? wl[i] : P::weight(L, q, base + i);
                if (x < run) { pick = i; break; }
            }
        } else if constexpr (S == WF_SAMPLER_ALIAS) {
            uint32_t x = q.rng.index(d);
            uint64_t k = q.rng.bits53();
            double split;
            uint32_t second;
            vose_bucket_local(d, sum, wl, x, split, second);
            pick = k < unit_threshold(split) ? x : second;
        } else {  // REJ over the gathered weights, p* = max
            uint32_t t = 0;
            for (;; ++t) {
                if (t >= L.trial_cap) {
                    raise_device(L, WF_ERR_REJECTION_CAP);
                    return kFault;
                }
                if (L.g.stats) atomicAdd(L.g.stats, 1ull);
                uint32_t x = q.rng.index(d);
                double y = q.rng.real(mx);
                if (y < P::weight(L, q, base + x)) { pick = x; break; }
            }
        }
    }
    if constexpr (P::needs_edge) edge = base + pick;
    if (F == kDirect && L.adj8) {
        // packed adjacency (dst, degree, base): one 8 B load
        uint64_t w;
        dst = adj8_unpack(ldr(reinterpret_cast<const uint64_t*>(L.adj8) + base + pick), L.adj8_vbits, L.adj8_dbits,
                          w);
        q.nb_word = w;
        q.have_nb = true;
        return kMoved;
    }
    if (F == kDirect && L.adj) {
        // decorated adjacency {dst, -, vertex word of dst}: one 16 B load
        uint4 a = ldr16(L.adj + base + pick);
        dst = a.x;
        q.nb_word = (static_cast<uint64_t>(a.w) << 32) | a.z;
        q.have_nb = true;
        return kMoved;
    }
    dst = ldr(L.g.nbr + base + pick);
    return kMoved;
}

// ---- warp-cooperative gather for hub vertices (gathered flows) -------------------
// gather (engine.hpp:134-184) evaluates weight(Q, e) over all d edges of the
// current vertex every step.  A lane doing that alone for a hub serialises d
// dependent loads (for Node2Vec each one an adjacency test) while its warp
// waits.  Instead, when a lane's current vertex has >= kCoopDegree edges, the
// whole warp evaluates its weights, 32 edges per round, and the lane samples
// from the result:
//   ITS   the pick is the first i with x < cumulative[i]: a warp-wide inclusive
//         scan per round of 32 weights, x drawn by the owner from its own stream;
//   ALIAS the weights go to the warp's scratch row; the owner runs Vose's
//         construction for its bucket over it (vose_bucket_staged, no re-evaluation);
//   REJ   p* = max weight (exact in any order); the owner runs the trials.
// Bit-exactness: the reference sums in edge order.  A reordered fp64 sum is
// the same number when every partial sum is exact, i.e. when all weights are
// multiples of a common power of two q and the total stays below 2^52 q (the
// survey checked this reordering for f32-valued weights).  Each
// step checks that certificate; without it ITS falls back to the owner's
// sequential scan and ALIAS sums the scratch row in edge order.  Dead ends
// (all weights zero) consume no draws; contract violations set the error word.
// Exponent of the lowest set bit of a positive finite double (its quantum).
__device__ __forceinline__ int quantum_exp(double w) {
    const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(w));
    const int e = static_cast<int>((b >> 52) & 0x7FF);
    const unsigned long long m = (b & 0xFFFFFFFFFFFFFull) | (e ? (1ull << 52) : 0ull);
    return (e ? e : 1) - 1075 + __ffsll(static_cast<long long>(m)) - 1;
}

// Node2Vec's gathered weights over a hub by a warp-wide merge of the sorted
// neighbour lists.  Every weight out of cur needs "is dst a neighbour of prev"
// (algorithms.hpp:103-119): over all of N(cur) that is the intersection
// N(cur) ∩ N(prev).  One adjacency test per edge is d random requests (a
// filter sector, then a hash bucket for ~6 %), and a warp waits for its
// slowest lane every round; the merge instead streams both lists in order,
// 128 entries at a time (coalesced loads), and each lane binary-searches its
// four cur-neighbours in the window of prev's list staged in shared memory.
// Same membership answers as Graph::has_edge on sorted adjacency (duplicates
// included), so the same weights, sums and draws.  Used when both lists are
// sorted and prev's list is at most kMergeRatio times cur's (else the per-edge
// tests read less).
constexpr uint32_t kMergeWin = 128;
constexpr uint32_t kMergeRatio = 8;

template <class F>
__device__ __forceinline__ void n2v_merge_weights(const WalkLaunch& L, const Walker& h, F&& emit) {
    __shared__ uint32_t merge_win[kBlock / 32][kMergeWin];
    constexpr uint32_t kPer = kMergeWin / 32;
    const int lane = threadIdx.x & 31;
    uint32_t* win = merge_win[threadIdx.x >> 5];
    const uint32_t* A = L.g.nbr + h.cur_base;
    const uint32_t* B = L.g.nbr + h.prev_base;
    const uint32_t d = h.cur_deg, dp = h.prev_deg;
    constexpr uint32_t kPast = 0xFFFFFFFFu;  // above every vertex id
    // the next window of prev's list and the next block of cur's are loaded
    // one step ahead (registers), so their round trips overlap the searches
    uint32_t bn[kPer], an[kPer];
    auto fetch_b = [&](uint32_t at) {
#pragma unroll
        for (uint32_t k = 0; k < kPer; ++k) {
            const uint32_t i = at + lane + 32 * k;
            bn[k] = i < dp ? __ldg(B + i) : kPast;
        }
    };
    auto fetch_a = [&](uint32_t at) {
#pragma unroll
        for (uint32_t k = 0; k < kPer; ++k) {
            const uint32_t i = at + lane + 32 * k;
            an[k] = i < d ? __ldg(A + i) : 0u;
        }
    };
    uint32_t ib = 0;
    auto next_window = [&]() {  // bn -> the window; prefetch the one after it
        __syncwarp();
#pragma unroll
        for (uint32_t k = 0; k < kPer; ++k) win[lane + 32 * k] = bn[k];
        __syncwarp();
        fetch_b(ib + kMergeWin);  // past the end: kPast, which closes any block
    };
    fetch_b(0);
    fetch_a(0);
    next_window();
    uint32_t bmax = win[kMergeWin - 1];
    unsigned long long windows = 1;
    for (uint32_t ia = 0; ia < d; ia += kMergeWin) {
        uint32_t a[kPer];
        bool found[kPer];
#pragma unroll
        for (uint32_t k = 0; k < kPer; ++k) {
            a[k] = an[k];
            found[k] = false;
        }
        // the block's largest entry (its last): lane off % 32, slot off / 32
        const uint32_t off = min(ia + kMergeWin, d) - 1 - ia;
        uint32_t mine = a[0];
#pragma unroll
        for (uint32_t k = 1; k < kPer; ++k) mine = k == off / 32 ? a[k] : mine;
        const uint32_t amax = __shfl_sync(kFull, mine, off & 31);
        if (ia + kMergeWin < d) fetch_a(ia + kMergeWin);
        for (;;) {
#pragma unroll
            for (uint32_t k = 0; k < kPer; ++k) {
                uint32_t lo = 0;  // lower_bound of a[k] in the window
#pragma unroll
                for (uint32_t s = kMergeWin / 2; s > 0; s >>= 1) lo = win[lo + s - 1] < a[k] ? lo + s : lo;
                found[k] = found[k] || (lo < kMergeWin && win[lo] == a[k]);
            }
            // prev's entries past this window are >= bmax: the block is done
            // once the window reaches its largest value
            if (bmax >= amax) break;
            ib += kMergeWin;
            next_window();
            bmax = win[kMergeWin - 1];
            ++windows;
        }
#pragma unroll
        for (uint32_t k = 0; k < kPer; ++k) {
            const uint32_t i = ia + lane + 32 * k;
            if (i < d) emit(i, a[k], found[k]);
        }
    }
    if (L.g.stats && lane == 0)  // instrumented runs: sectors of prev's list streamed
        atomicAdd(L.g.stats + 1, windows * (kMergeWin * 4 / 32));
}

template <class P, int S>
__device__ __forceinline__ void coop_step(const WalkLaunch& L, Walker& q, int leader, double* wrow_warp) {
    const int lane = threadIdx.x & 31;
    Walker h = q;  // the owner's walker, as every lane sees it
    h.row = __shfl_sync(kFull, q.row, leader);
    h.cur = __shfl_sync(kFull, q.cur, leader);
    h.prev = __shfl_sync(kFull, q.prev, leader);
    h.cur_base = __shfl_sync(kFull, q.cur_base, leader);
    h.prev_base = __shfl_sync(kFull, q.prev_base, leader);
    h.cur_deg = __shfl_sync(kFull, q.cur_deg, leader);
    h.prev_deg = __shfl_sync(kFull, q.prev_deg, leader);
    h.len = __shfl_sync(kFull, q.len, leader);
    const uint32_t d = h.cur_deg;
    const uint64_t base = h.cur_base;
    double* wrow = wrow_warp;  // the warp's row: weights (ITS, ALIAS) + Vose's park area (ALIAS)
    if (L.g.stats && lane == leader) atomicAdd(L.g.stats + 2, static_cast<unsigned long long>(d));
    // pass 1: weights, validity, partial sums, max, smallest quantum; for
    // ALIAS also the positive weights' count and smallest value and the rank
    // of bucket x (drawn next, peeked now) among the zero / positive weights
    double lsum = 0.0, lmax = 0.0;
    int qexp = 0x7FFFFFFF;
    bool bad = false;
    bool merged = false;
    uint32_t xpeek = 0, npos = 0, nbefore = 0;
    double pmin = 1.7976931348623157e308;
    if constexpr (S == WF_SAMPLER_ALIAS) {
        if (lane == leader) xpeek = static_cast<uint32_t>(__umul64hi(q.rng.peek(), static_cast<uint64_t>(d)));
        xpeek = __shfl_sync(kFull, xpeek, leader);
    }
    auto alias_stats = [&](uint32_t i, double w) {
        if constexpr (S == WF_SAMPLER_ALIAS) {
            if (w > 0.0) {
                ++npos;
                pmin = w < pmin ? w : pmin;
                nbefore += i < xpeek;
            }
        }
    };
    if constexpr (P::kind == WF_PROGRAM_NODE2VEC) {
        if (h.len > 1 && L.g.sorted && h.prev_deg <= kMergeRatio * d) {
            const ProgParams& p = L.prog;
            n2v_merge_weights(L, h, [&](uint32_t i, uint32_t dst, bool common) {
                double w = dst == h.prev ? p.inv_a : common ? 1.0 : p.inv_b;
                if (p.weighted) w = __dmul_rn(w, edge_weight(L.g, base + i));
                if (!(w >= 0.0 && w <= 1.7976931348623157e308)) bad = true;
                if (S == WF_SAMPLER_ALIAS || (S == WF_SAMPLER_ITS && wrow)) wrow[i] = w;
                if (w > 0.0) qexp = min(qexp, quantum_exp(w));
                lsum += w;
                lmax = w > lmax ? w : lmax;
                alias_stats(i, w);
            });
            merged = true;
        }
    }
    if (!merged) {
        // eight 32-edge rounds per batch: their weight loads are issued
        // together, ahead of the row stores
        constexpr int kR = 8;
        for (uint32_t c0 = 0; c0 < d; c0 += 32 * kR) {
            double wv[kR];
#pragma unroll
            for (int r = 0; r < kR; ++r) {
                const uint32_t i = c0 + 32 * r + lane;
                wv[r] = i < d ? P::weight(L, h, base + i) : 0.0;
            }
#pragma unroll
            for (int r = 0; r < kR; ++r) {
                const uint32_t i = c0 + 32 * r + lane;
                if (i >= d) break;
                const double w = wv[r];
                if (!(w >= 0.0 && w <= 1.7976931348623157e308)) bad = true;
                if (S == WF_SAMPLER_ALIAS || (S == WF_SAMPLER_ITS && wrow)) wrow[i] = w;
                if (w > 0.0) qexp = min(qexp, quantum_exp(w));
                lsum += w;
                lmax = w > lmax ? w : lmax;
                alias_stats(i, w);
            }
        }
    }
    if (__any_sync(kFull, bad)) {  // check_program_weight (engine.hpp:97-101)
        if (lane == leader) {
            raise_device(L, WF_ERR_CONTRACT);
            q.coop = kCoopFault;
        }
        return;
    }
    double sum = lsum, mx = lmax;
    for (int o = 16; o > 0; o >>= 1) {
        sum += __shfl_xor_sync(kFull, sum, o);
        const double m2 = __shfl_xor_sync(kFull, mx, o);
        mx = m2 > mx ? m2 : mx;
        qexp = min(qexp, __shfl_xor_sync(kFull, qexp, o));
    }
    if (!(sum > 0.0)) {  // all weights zero (exact in any order): dead end, no draws
        if (lane == leader) q.coop = kCoopDead;
        return;
    }
    // every partial sum a multiple of 2^qexp below 2^52 * 2^qexp: exact
    const bool exact = sum < ldexp(1.0, 52 + max(qexp, -1000));
    if constexpr (S == WF_SAMPLER_ITS) {
        if (!exact) return;  // the owner scans sequentially in move()
        double x = 0.0;
        if (lane == leader) x = q.rng.real(sum);  // == cumulative[d-1]
        x = __shfl_sync(kFull, x, leader);
        // pass 2: first i with x < cumulative[i] (engine.hpp:373-377)
        double running = 0.0;
        uint32_t pick = d - 1;
        if (wrow) __syncwarp();  // pass 1's weights are in the row
        // with the row: eight 32-weight rounds loaded at once, so a hub's scan
        // waits on one load round trip per 256 weights instead of per 32; a
        // batch that ends below x is skipped on its total (one warp
        // reduction) — only the batch holding the pick is scanned round by
        // round.  Every partial sum is exact (the certificate), so the
        // reordered totals are the cumulative sums the reference compares.
        constexpr uint32_t kG = 8;
        for (uint32_t c0 = 0; wrow && c0 < d; c0 += 32 * kG) {
            double v[kG];
#pragma unroll
            for (uint32_t k = 0; k < kG; ++k) {
                const uint32_t i = c0 + 32 * k + lane;
                v[k] = i < d ? wrow[i] : 0.0;
            }
            double tot = 0.0;
#pragma unroll
            for (uint32_t k = 0; k < kG; ++k) tot += v[k];
            for (int o = 16; o > 0; o >>= 1) tot += __shfl_xor_sync(kFull, tot, o);
            if (!(x < running + tot) && c0 + 32 * kG < d) {
                running += tot;
                continue;
            }
            bool hit_any = false;
#pragma unroll
            for (uint32_t k = 0; k < kG; ++k) {
                const uint32_t c = c0 + 32 * k;
                if (c >= d) break;
                double s = v[k];
                for (int o = 1; o < 32; o <<= 1) {  // inclusive scan (exact)
                    const double u = __shfl_up_sync(kFull, s, o);
                    if (lane >= o) s += u;
                }
                const unsigned hit = __ballot_sync(kFull, c + lane < d && x < running + s);
                if (hit) {
                    pick = c + __ffs(hit) - 1;
                    hit_any = true;
                    break;
                }
                running += __shfl_sync(kFull, s, 31);
            }
            if (hit_any) break;
        }
        for (uint32_t c = 0; !wrow && c < d; c += 32) {
            const uint32_t i = c + lane;
            // no row (pass 1's weights were not kept): evaluated again
            double v = i < d ? P::weight(L, h, base + i) : 0.0;
            for (int o = 1; o < 32; o <<= 1) {  // inclusive scan (exact)
                const double u = __shfl_up_sync(kFull, v, o);
                if (lane >= o) v += u;
            }
            const unsigned hit = __ballot_sync(kFull, i < d && x < running + v);
            if (hit) {
                pick = c + __ffs(hit) - 1;
                break;
            }
            running += __shfl_sync(kFull, v, 31);
        }
        if (lane == leader) {
            q.coop = kCoopPick;
            q.coop_pick = pick;
        }
        if (wrow) __syncwarp();  // the row is free for the next hub
    } else if constexpr (S == WF_SAMPLER_ALIAS) {
        __syncwarp();  // the scratch row is complete
        double total = sum;
        if (!exact) {  // the reference's edge-order sum, by the owner
            double seq = 0.0;
            if (lane == leader)
                for (uint32_t i = 0; i < d; ++i) seq += wrow[i];
            total = __shfl_sync(kFull, seq, leader);
        }
        uint32_t x = 0;
        uint64_t k = 0;
        if (lane == leader) {
            x = q.rng.index(d);
            k = q.rng.bits53();
        }
        x = __shfl_sync(kFull, x, leader);
        double split;
        uint32_t second;
        for (int o = 16; o > 0; o >>= 1) {
            npos += __shfl_xor_sync(kFull, npos, o);
            nbefore += __shfl_xor_sync(kFull, nbefore, o);
            const double m2 = __shfl_xor_sync(kFull, pmin, o);
            pmin = m2 < pmin ? m2 : pmin;
        }
        // every positive weight the same (MetaPath's 0/1, unweighted programs):
        // the replay has a closed form (vose_bucket_uniform), else the chain
        const uint32_t xi = (x & ~31u) | static_cast<uint32_t>(lane);
        const bool xpos = __shfl_sync(kFull, xi < d ? wrow[xi] : 0.0, x & 31) > 0.0;
        const uint32_t xrank = xpos ? nbefore : x - nbefore;
        if (!(pmin == mx && vose_bucket_uniform(d, npos, mx, total, x, xpos, xrank, wrow, split, second)))
            vose_bucket_staged(d, wrow, total, x, wrow + L.scratch_stride, split, second);
        if (lane == leader) {
            q.coop = kCoopPick;
            q.coop_pick = k < unit_threshold(split) ? x : second;
        }
        __syncwarp();  // the row is free for the next hub
    } else {  // REJ over the gathered weights, p* = max (sampler.hpp:152-164)
        if (lane == leader) {
            for (uint32_t t = 0;; ++t) {
                if (t >= L.trial_cap) {
                    raise_device(L, WF_ERR_REJECTION_CAP);
                    q.coop = kCoopFault;
                    return;
                }
                if (L.g.stats) atomicAdd(L.g.stats, 1ull);
                const uint32_t x = q.rng.index(d);
                const double y = q.rng.real(mx);
                if (y < P::weight(L, q, base + x)) {
                    q.coop = kCoopPick;
                    q.coop_pick = x;
                    return;
                }
            }
        }
    }
}

// Whether a gathered launch takes the cooperative hub path (MetaPath's
// label-index ITS needs no gather at all).
template <class P, int S, int F>
__device__ __forceinline__ bool coop_gathered(const WalkLaunch& L) {
    if constexpr (F != kGathered) return false;
    if constexpr (P::kind == WF_PROGRAM_METAPATH && S == WF_SAMPLER_ITS) return !L.use_label_index;
    return true;
}

// Loads what the next move out of q.cur needs into registers.
template <class P, int S, int F>
__device__ __forceinline__ void load_current(const WalkLaunch& L, Walker& q) {
    if constexpr (P::kind == WF_PROGRAM_METAPATH && S == WF_SAMPLER_ITS && F == kGathered) {
        if (L.use_label_index) {
            const uint4* rec = L.g.lab_rec + 2 * static_cast<uint64_t>(q.cur);
            uint4 r0, r1;
            ldr256(rec, r0, r1);
            uint64_t base = (static_cast<uint64_t>(r0.y) << 32) | r0.x;
            uint32_t ends[kMaxIndexedLabels] = {r0.z, r0.w, r1.x, r1.y, r1.z, r1.w};
            uint32_t l = __ldg(L.prog.schema + (q.len - 1));
            uint32_t lo = 0, hi = 0;
#pragma unroll
            for (int i = 0; i < kMaxIndexedLabels; ++i) {
                if (static_cast<uint32_t>(i) == l) hi = ends[i];
                if (static_cast<uint32_t>(i) + 1 == l) lo = ends[i];
            }
            if (l >= static_cast<uint32_t>(kMaxIndexedLabels)) lo = hi = 0;
            q.cur_base = base + lo;
            q.cur_deg = hi - lo;
            return;
        }
    }
    decode_vertex(L.g, L.sview, q.cur, q.cur_base, q.cur_deg);
}

// True when load_current is a plain vertex-word read (everything but
// MetaPath's label-index flow), which can then be deferred (Walker::pend).
template <class P, int S, int F>
__device__ __forceinline__ bool plain_word(const WalkLaunch& L) {
    if constexpr (P::kind == WF_PROGRAM_METAPATH && S == WF_SAMPLER_ITS && F == kGathered) return !L.use_label_index;
    return true;
}

// What load_current would read for a walk starting at `src`, packed as a
// vertex word (base << 24 | deg) for claim-time staging; kNoWord when it does
// not pack (a label group of >= 2^24 - 1 edges): that lane loads it itself.
constexpr unsigned long long kNoWord = ~0ull;
template <class P, int S, int F>
__device__ __forceinline__ unsigned long long start_word(const WalkLaunch& L, uint32_t src) {
    if constexpr (P::kind == WF_PROGRAM_METAPATH && S == WF_SAMPLER_ITS && F == kGathered) {
        if (L.use_label_index) {
            uint4 r0, r1;
            ldr256(L.g.lab_rec + 2 * static_cast<uint64_t>(src), r0, r1);
            const uint64_t base = (static_cast<uint64_t>(r0.y) << 32) | r0.x;
            const uint32_t ends[kMaxIndexedLabels] = {r0.z, r0.w, r1.x, r1.y, r1.z, r1.w};
            const uint32_t l = __ldg(L.prog.schema);
            uint32_t lo = 0, hi = 0;
#pragma unroll
            for (int i = 0; i < kMaxIndexedLabels; ++i) {
                if (static_cast<uint32_t>(i) == l) hi = ends[i];
                if (static_cast<uint32_t>(i) + 1 == l) lo = ends[i];
            }
            if (l >= static_cast<uint32_t>(kMaxIndexedLabels)) lo = hi = 0;
            const uint64_t gb = base + lo;
            const uint32_t cnt = hi - lo;
            return cnt < kDegEscape && gb < (1ull << 40) ? (gb << kDegBits) | cnt : kNoWord;
        }
    }
    return ldr(L.sview + src);
}

template <bool ST>
__device__ __forceinline__ uint32_t source_at(const WalkLaunch& L, uint64_t qid) {  // walker.hpp:70-77
    if (L.qmode == WF_QUERY_ONE_PER_VERTEX) return static_cast<uint32_t>(qid);
    if (L.qmode == WF_QUERY_FROM_SOURCE) return L.qsource;
    if constexpr (ST) {
        // L2 only, ordered after wait_sources: the list lands while the
        // kernel runs
        uint32_t v;
        asm volatile("ld.global.cg.u32 %0, [%1];" : "=r"(v) : "l"(L.qsources + qid) : "memory");
        return v;
    }
    return __ldg(L.qsources + qid);
}

// Path rows are written whole 32 B sectors at a time: each lane stages its
// next kPathGroup vertices in shared memory ([slot][thread], conflict-free)
// and stores them with 256-bit stores when the group fills or the walk ends.
// Single 4 B stores to 32 B-strided rows made every step a partial-sector
// write (ncu: 4x the algorithmic DRAM write bytes).  Used when rows are
// 32 B-aligned (stride % 8 == 0); otherwise one 4 B store per vertex.
#ifndef WF_PATH_GROUP
#define WF_PATH_GROUP 8
#endif
constexpr uint32_t kPathGroup = WF_PATH_GROUP;  // 8, 16 or 32 vertices
struct PathStage {
    uint32_t* s;  // kBlock * kPathGroup words
    __device__ __forceinline__ uint32_t& at(uint32_t slot) { return s[slot * kBlock + threadIdx.x]; }
};

// One 256-bit store (st.global.v8, sm_100) of staged words [8k, 8k + 8).
__device__ __forceinline__ void store_sector(uint32_t* dst, PathStage ps, uint32_t k) {
    const uint32_t b = 8 * k;
#ifdef WF_PATH_EVICT_LAST
    // experiment: evict-last L2 policy on the path sectors (their line fills
    // over four groups)
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    asm volatile("st.global.L2::cache_hint.v8.u32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8}, %9;" ::"l"(dst + b),
                 "r"(ps.at(b)), "r"(ps.at(b + 1)), "r"(ps.at(b + 2)), "r"(ps.at(b + 3)), "r"(ps.at(b + 4)),
                 "r"(ps.at(b + 5)), "r"(ps.at(b + 6)), "r"(ps.at(b + 7)), "l"(pol)
                 : "memory");
    return;
#endif
    asm volatile("st.global.v8.u32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(dst + b), "r"(ps.at(b)),
                 "r"(ps.at(b + 1)), "r"(ps.at(b + 2)), "r"(ps.at(b + 3)), "r"(ps.at(b + 4)), "r"(ps.at(b + 5)),
                 "r"(ps.at(b + 6)), "r"(ps.at(b + 7))
                 : "memory");
}

// The first `nsec` sectors of a lane's staged group.
__device__ __forceinline__ void store_group(uint32_t* dst, PathStage ps, uint32_t nsec = kPathGroup / 8) {
#pragma unroll
    for (uint32_t k = 0; k < kPathGroup / 8; ++k)
        if (k < nsec) store_sector(dst, ps, k);
}

__device__ __forceinline__ void finish(const WalkLaunch& L, const Walker& q, int st, PathStage ps) {
#ifdef WF_DIAG_FINISH_TIME
    // diagnostic builds only (tools/profile_walk.py --diag-times): the walk's
    // completion time in 32 ns units (low 24 bits) and min(length, 255)
    // replace its length
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    L.lengths[q.row] = (static_cast<uint32_t>(t >> 5) << 8) | min(q.len, 255u);
#else
    L.lengths[q.row] = q.len;
#endif
    L.status[q.row] = static_cast<uint8_t>(st);
    if (L.staged) {
        // the open group as whole-sector stores (words past the length are
        // unspecified row padding, as the rest of the row)
        const uint32_t g0 = q.len & ~(kPathGroup - 1);
        const uint32_t end = min(q.len, L.stride);
        if (g0 < end) store_group(L.paths + q.row * L.stride + g0, ps, (end - g0 + 7) / 8);
    }
    if (q.len > L.stride) atomicAdd(L.overflow_out, 1ULL);
}

// Host streaming: `rows` finished rows of tile `tile` carrying `verts`
// vertices (one call per tile per warp iteration).  Callers have fenced their
// row / length / status stores, so a published chunk is complete in memory
// for the compaction kernel the host queues on seeing its flag.
constexpr int kCountShift = 40;
constexpr unsigned long long kSumMask = (1ull << kCountShift) - 1;
static __device__ __noinline__ void stream_report(unsigned long long* tile_word, unsigned long long* chunk_word,
                                           unsigned long long* chunk_flag, uint64_t n_rows,
                                           uint32_t shifts, uint32_t tile, uint32_t rows, uint32_t verts) {
    const uint32_t tile_shift = shifts & 0xFF, chunk_tiles_shift = shifts >> 8;
    const unsigned long long add = (static_cast<unsigned long long>(rows) << kCountShift) | verts;
    const unsigned long long now = atomicAdd(tile_word + tile, add) + add;
    const uint64_t t0 = static_cast<uint64_t>(tile) << tile_shift;
    const uint64_t tile_rows = min(static_cast<uint64_t>(1) << tile_shift, n_rows - t0);
    if ((now >> kCountShift) != tile_rows) return;
    // this report completed the tile: add it to its chunk
    __threadfence();
    const uint32_t chunk = tile >> chunk_tiles_shift;
    const uint64_t ntiles = (n_rows + (1ull << tile_shift) - 1) >> tile_shift;
    const uint64_t c0 = static_cast<uint64_t>(chunk) << chunk_tiles_shift;
    const uint64_t chunk_tiles = min(static_cast<uint64_t>(1) << chunk_tiles_shift, ntiles - c0);
    const unsigned long long cadd = (1ull << kCountShift) | (now & kSumMask);
    const unsigned long long cnow = atomicAdd(chunk_word + chunk, cadd) + cadd;
    if ((cnow >> kCountShift) != chunk_tiles) return;
    // ... and the chunk: publish its vertex total to the host
    __threadfence_system();
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(chunk_flag + chunk), "l"((cnow & kSumMask) + 1)
                 : "memory");
}
__device__ __forceinline__ void stream_report(const WalkLaunch& L, uint32_t tile, uint32_t rows, uint32_t verts) {
    stream_report(L.tile_word, L.chunk_word, L.chunk_flag, L.n_rows, L.tile_shift | (L.chunk_tiles_shift << 8),
                  tile, rows, verts);
}

// Host streaming: wait until the source list holds rows [0, need) (the copy
// stream writes src_ready behind each block's copy).  Bounded: a copy that
// never lands raises a device error instead of hanging the GPU.
// Returns the rows known resident.
static __device__ __noinline__ uint64_t wait_sources(const unsigned int* src_ready, uint32_t src_shift, int* error_word,
                                              uint64_t need) {
    unsigned long long t0, t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (;;) {
        unsigned int r;
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(r) : "l"(src_ready) : "memory");
        const uint64_t have = static_cast<uint64_t>(r) << src_shift;
        if (have >= need) return have;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        if (t - t0 > 10000000000ull) {  // 10 s
            atomicCAS(error_word, 0, WF_ERR_CUDA);
            return ~0ull;
        }
        __nanosleep(200);
    }
}

__device__ __forceinline__ void emit(const WalkLaunch& L, const Walker& q, uint32_t p, uint32_t v,
                                     PathStage ps) {
    if (p < L.stride) {
        if (L.staged) {
            const uint32_t slot = p & (kPathGroup - 1);
            ps.at(slot) = v;
            if (slot == kPathGroup - 1) store_group(L.paths + q.row * L.stride + (p - slot), ps);
        } else {
            L.paths[q.row * L.stride + p] = v;
        }
    }
    // In-kernel: these atomics overlap the walk's load latency.  Counting the
    // rows in a pass after the kernel measured slower (C2: 0.29 vs 0.25 ms).
    if (L.visit_counts) atomicAdd(L.visit_counts + v, 1u);
}

// The persistent step kernel.  One walker per lane; lanes whose walk ended take
// the next row from their warp's claimed block of rows (the GPU analogue of the
// interleaved executor's admit/refill, interleave.hpp:436-464, 531-538), so
// PPR's geometric terminations never idle a lane while queries remain.  Every
// walker draws only from its own (seed, qid) stream, so the output is
// independent of scheduling, exactly as in the reference.
//
// Register bound: 8 x 256 threads per SM (<= 32 registers) for the flows whose
// state fits it; the launch tuner (wf_session_tune) may run fewer blocks.  The
// gathered flows (per-step scans, on-the-fly Vose) keep their registers.
// Build knobs (experiments only): WF_BLOCK, WF_MIN_BLOCKS, WF_N2V_BLOCKS,
// WF_CLAIM (128-thread blocks measured the same as 256).
template <class P, int S, int F>
constexpr int walk_min_blocks() {
    // Node2Vec's O-REJ step (edge hash probe) needs ~48 registers without
    // spills (5 blocks: 23.9 vs 22.9 G steps/s at 6 with 76 B of spills, C3);
    // MetaPath's label-index ITS path is the C4 hot loop (its generic
    // gathered fallback shares the kernel).
#ifndef WF_MIN_BLOCKS
#define WF_MIN_BLOCKS 4
#endif
    if (F == kGathered) return (P::kind == WF_PROGRAM_METAPATH && S == WF_SAMPLER_ITS) ? WF_MIN_BLOCKS : 1;
#ifndef WF_N2V_BLOCKS
#define WF_N2V_BLOCKS 5
#endif
    return P::kind == WF_PROGRAM_NODE2VEC ? WF_N2V_BLOCKS : WF_MIN_BLOCKS;
}

// Rows a warp claims from the global cursor per atomic.  One atomic per refill
// put every warp's refill on one L2 address (~every other iteration for PPR):
// C4 15.9 -> 31.7 G steps/s, C5 33.5 -> 40.5 G with 32-row claims.
#ifndef WF_CLAIM
#define WF_CLAIM 32
#endif
constexpr uint32_t kClaim = WF_CLAIM;

// ST: the host-streaming instantiation (run_to_host): the source list may
// land during the run (src_ready) and, when tile_word is set, finished rows
// report to their tile / chunk words.
// A separate instantiation keeps the device-output kernels' registers as they
// were (the reports cost ~10 registers, which would cost C3/C5 a block/SM).
template <class P, int S, int F, bool ST>
__global__ void __launch_bounds__(kBlock, walk_min_blocks<P, S, F>()) walk_kernel(const WalkLaunch L) {
    const int lane = threadIdx.x & 31;
    __shared__ uint32_t stage_words[kPathGroup * kBlock];
    PathStage ps{stage_words};
    Walker q;
    q.row = 0;
    q.cur = q.prev = 0;
    q.cur_deg = q.prev_deg = 0;
    q.cur_base = q.prev_base = 0;
    q.len = 0;
    q.trials = 0;
    q.rng.s = 0;
    q.nb_word = 0;
    q.have_nb = false;
    q.pend = false;
    q.coop = kCoopNone;
    q.coop_pick = 0;
    bool active = false;
    bool fresh = false;
    bool drained = false;
    // warp-uniform claim state, kept in shared memory (registers are the
    // occupancy limit of the O-REJ kernels): next unstarted row of the warp's
    // claimed block and the rows left in it
    __shared__ unsigned long long claim_next[kBlock / 32];
    __shared__ uint32_t claim_left[kBlock / 32];
    // Claim-time staging: the sources of the claimed rows and their vertex
    // words are loaded by the whole warp at once (one coalesced load + one
    // gather per 32 rows) into shared memory, so a refilled lane moves in the
    // same iteration instead of sitting one out on its own source -> word load
    // chain (C1 -5 %, C5 -1.6 %; and no register spills).  For MetaPath's
    // label index the staged word is the source's first label group.
    __shared__ unsigned long long claim_first[kBlock / 32];
    __shared__ uint32_t claim_src[kBlock / 32][kClaim];
    __shared__ unsigned long long claim_word[kBlock / 32][kClaim];
    const int wid = threadIdx.x >> 5;
    // A static prefix of the rows is dealt to the warps in kClaim-row blocks,
    // round robin (block k of warp w = k * warps + w), without the cursor
    // atomic whose round trip was the refill's top stall (ncu, C2); the rest
    // is claimed through the cursor for balance.
    __shared__ uint32_t claim_k[kBlock / 32];
    // host streaming: source rows this warp has seen resident
    __shared__ unsigned long long src_seen[kBlock / 32];
    if (lane == 0) {
        claim_next[wid] = 0;
        claim_left[wid] = 0;
        claim_k[wid] = 0;
        src_seen[wid] = 0;
    }
    __syncwarp();
    unsigned long long steps = 0;
    for (;;) {
        // refill lanes without a live walker from the warp's claimed block of rows
        for (;;) {
            unsigned need = __ballot_sync(kFull, !active && !drained);
            if (need == 0) break;
            uint64_t wnext = claim_next[wid];
            uint32_t wleft = claim_left[wid];
            if (wleft == 0) {
                const uint32_t nwarps = gridDim.x * (kBlock / 32);
                const uint32_t k = claim_k[wid];
                if (k < L.static_blocks) {
                    wnext = (static_cast<uint64_t>(k) * nwarps + blockIdx.x * (kBlock / 32) + wid) * kClaim;
                    wleft = kClaim;
                    __syncwarp();
                    if (lane == 0) claim_k[wid] = k + 1;
                } else {
                // guided claim: up to kClaim rows while the queue is long,
                // shrinking to the lanes in need near its end (balance)
                const uint64_t at = wnext > L.dyn_base ? wnext : L.dyn_base;
                const uint64_t est = at < L.n_rows ? L.n_rows - at : 0;
                const uint64_t share = est / (2ull * nwarps);
                const uint32_t want = max(static_cast<uint32_t>(__popc(need)),
                                          share < kClaim ? static_cast<uint32_t>(share) : kClaim);
                unsigned long long first = 0;
                if (lane == 0) first = atomicAdd(L.cursor, static_cast<unsigned long long>(want));
                first = __shfl_sync(kFull, first, 0) + L.dyn_base;
                wnext = first;
                const uint64_t rest = first >= L.n_rows ? 0 : L.n_rows - first;
                wleft = rest < want ? static_cast<uint32_t>(rest) : want;
                }
                if (wleft == 0) {  // queue drained: every idle lane is done
                    drained = drained || !active;
                    continue;
                }
                if (ST && L.src_ready && wnext + wleft > src_seen[wid]) {
                    if (lane == 0) {
                        const uint64_t have =
                            wait_sources(L.src_ready, L.src_shift, L.error_word, L.src_row0 + wnext + wleft);
                        src_seen[wid] = have == ~0ull ? have : have - L.src_row0;
                    }
                    __syncwarp();
                }
                {
                    uint32_t src = 0;
                    unsigned long long word = 0;
                    if (static_cast<uint32_t>(lane) < wleft) {
                        const uint64_t qid = L.qid_map ? __ldg(L.qid_map + wnext + lane) : L.qid_begin + wnext + lane;
                        src = source_at<ST>(L, qid);
                        if (src < L.g.V) word = start_word<P, S, F>(L, src);
                    }
                    claim_src[wid][lane] = src;
                    claim_word[wid][lane] = word;
                    if (lane == 0) claim_first[wid] = wnext;
                    __syncwarp();
                }
            }
            const uint32_t rank = __popc(need & ((1u << lane) - 1));
            const uint32_t take = min(static_cast<uint32_t>(__popc(need)), wleft);
            __syncwarp();
            if (lane == 0) {
                claim_next[wid] = wnext + take;
                claim_left[wid] = wleft - take;
            }
            __syncwarp();
            if (!active && !drained && rank < take) {
                const uint64_t row = wnext + rank;
                const uint64_t qid = L.qid_map ? __ldg(L.qid_map + row) : L.qid_begin + row;
                q.row = row;
                q.rng.s = stream_state(L.seed_mixed, qid);
                const uint32_t slot = static_cast<uint32_t>(row - claim_first[wid]);
                q.cur = claim_src[wid][slot];
                q.prev = 0xFFFFFFFFu;
                q.len = 0;
                q.trials = 0;
                if (q.cur >= L.g.V) {
                    // QuerySpec validation (walker.cpp:8-109) on the device: the
                    // run reports ConfigError (its rows are not results)
                    raise_device(L, WF_ERR_CONFIG);
                    q.cur = 0;
                }
                {
                    emit(L, q, 0, q.cur, ps);
                    q.len = 1;
                    if (P::prechecked && P::finished(L, q)) {
                        finish(L, q, WF_WALK_COMPLETE, ps);  // walk_already_finished, program.hpp:86-93
                        if (ST && L.tile_word) {
                            __threadfence();
                            stream_report(L, static_cast<uint32_t>(row >> L.tile_shift), 1, 1);
                        }
                    } else {
                        const unsigned long long w = claim_word[wid][slot];
                        active = true;
                        if (w != kNoWord) {
                            if constexpr (kDeferWord<P>) {
                                q.nb_word = w;
                                q.pend = true;
                            } else {
                                unpack_word(L.g, w, q.cur, q.cur_base, q.cur_deg);
                            }
                        } else {
                            load_current<P, S, F>(L, q);
                            fresh = true;
                        }
                    }
                }
            }
        }
        if (!__any_sync(kFull, active)) break;
        // A lane whose start could not be staged (a label group too large for
        // a packed word) sits one iteration out: its load is still in flight,
        // and consuming it now would stall the whole warp on that load.
        const bool ready = active && !fresh;
        fresh = false;
        if constexpr (F == kGathered) {
            if (coop_gathered<P, S, F>(L)) {
                if constexpr (kDeferWord<P>) {
                    if (ready && q.pend) {
                        unpack_word(L.g, q.nb_word, q.cur, q.cur_base, q.cur_deg);
                        q.pend = false;
                    }
                }
                // hub steps of this warp, one after the other, by the whole warp
                unsigned hubs = __ballot_sync(kFull, ready && q.cur_deg >= kCoopDegree);
                double* wrow = L.scratch ? L.scratch + ((blockIdx.x * static_cast<uint64_t>(kBlock) + threadIdx.x) >> 5) *
                                                           (2 * L.scratch_stride)
                                         : nullptr;
                while (hubs) {
                    const int leader = __ffs(hubs) - 1;
                    hubs &= hubs - 1;
                    coop_step<P, S>(L, q, leader, wrow);
                }
            }
        }
        if (ready) {
            uint32_t dst = 0;
            uint64_t edge = 0;
            int r = move<P, S, F>(L, q, dst, edge);
            if (r == kMoved) {
                q.prev = q.cur;
                q.prev_base = q.cur_base;
                q.prev_deg = q.cur_deg;
                q.cur = dst;
                const uint32_t p = q.len;
                q.len += 1;
                steps += 1;
                // update (PPR's stop coin) before the path store: its draw
                // overlaps the neighbour load the store waits for (Node2Vec,
                // with kDeferWord off, keeps its original order)
                bool done;
                if constexpr (P::kind == WF_PROGRAM_NODE2VEC) {
                    emit(L, q, p, dst, ps);
                    done = P::update(L, q, edge);
                } else {
                    done = P::update(L, q, edge);
                    emit(L, q, p, dst, ps);
                }
                if (done) {
                    finish(L, q, WF_WALK_COMPLETE, ps);
                    active = false;
                } else if (q.have_nb) {
                    // unpacked by the next move (kDeferWord)
                    if constexpr (kDeferWord<P>) q.pend = true;
                    else unpack_word(L.g, q.nb_word, q.cur, q.cur_base, q.cur_deg);
                } else if (kDeferWord<P> && plain_word<P, S, F>(L)) {
                    q.nb_word = ldr(L.sview + q.cur);
                    q.pend = true;
                } else {
                    load_current<P, S, F>(L, q);
                }
                q.have_nb = false;
            } else if (r != kRetry) {
                finish(L, q, WF_WALK_DEAD_END, ps);
                active = false;
            }
        }
        if (ST && L.tile_word) {
            // host streaming: the rows finished this iteration report to their
            // tiles, one atomic per tile per warp
            const bool f = ready && !active;
            unsigned fm = __ballot_sync(kFull, f);
            if (fm) {
                // the finished rows' stores are ordered before each leader's
                // release (warp barrier, then a release fence: cumulative over
                // what the barrier made it observe)
                __syncwarp();
                const uint32_t tile = static_cast<uint32_t>(q.row >> L.tile_shift);
                do {  // usually one round: a warp's rows come from one or two tiles
                    const int leader = __ffs(fm) - 1;
                    const uint32_t lt = __shfl_sync(kFull, tile, leader);
                    const bool mine = f && tile == lt;
                    const unsigned grp = __ballot_sync(kFull, mine);
                    const uint32_t verts = __reduce_add_sync(kFull, mine ? q.len : 0u);
                    if (lane == leader) {
                        asm volatile("fence.acq_rel.gpu;" ::: "memory");
                        stream_report(L, lt, __popc(grp), verts);
                    }
                    fm &= ~grp;
                } while (fm);
            }
        }
    }
    // one atomic per warp for the step total
    for (int o = 16; o > 0; o >>= 1) steps += __shfl_xor_sync(kFull, steps, o);
    if (lane == 0 && steps) atomicAdd(L.steps_out, steps);
}

}  // namespace wf
