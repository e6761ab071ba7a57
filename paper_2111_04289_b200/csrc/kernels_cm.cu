// Cluster Monitoring aggregate pass (CM1S/CM1T, CM2S): newline framing + field decode +
// validation + predicate + warp-ballot compaction + pane partial aggregation.
//
// PAPER.md: Table IV CM1 "SUM(cpu) ... GROUPBY category ORDERBY SUM(cpu)", CM2
// "AVG(cpu) ... WHERE (eventType == 1) GROUPBY jobId"; record size "130 ~ 145 B (per record,
// variable)"; operators Scan (CSV) / Filtering / Projection / Aggregation (Table III).
// Record grammar: DESIGN.md reading R1 (13-column task_events line, <= 255 B + '\n').
//
// Design (B200).  Persistent CTAs of 4 warps, 5 CTAs per SM.  Every WARP walks its own
// contiguous range of warp tiles through a private 2-stage smem ring filled by TMA-engine bulk
// copies (cp.async.bulk, L2 evict-first), so no CTA barrier sits in the loop.  A warp tile is a
// 4352 B window = 4096 B payload + 256 B right halo (the tail of the last record that STARTS in
// the payload: a record belongs to the tile holding its first byte) + a 16 B left halo (the
// byte before the tile).  The producer (lane 0) issues a tile two tiles ahead and packs its
// geometry into one register word; every lane waits on the stage's mbarrier.
//  * Pass 1 (lane l: 32 B words l, l+32, ...; conflict-free LDS.128): exact SWAR byte equality
//    against '\n' and ',' (3 ops per 4-byte word and class), gathered to one mask bit per byte
//    with IDP.4A chains; the masks go to per-warp smem.  The right halo's masks are the next
//    tile's first 256 B: carried over, so a tile classifies exactly 4096 new bytes.
//  * Pass 2: lane l owns payload chunk l (128 B); records are owned by the '\n' before them;
//    a record's '\n' is the first one of chunk l+1 or l+2 (shuffles, branch-free first-bit).
//  * Pass 3, per record (one per lane per round, branch-free fast path cm_fast for the usual
//    shape): the 12 commas are pinned by bit tests in a 64-bit head window at the record start
//    and a 64-bit tail window ending at the '\n', plus zero tests of the windows between them;
//    ts / jobId / cpu digits are validated and valued with SWAR arithmetic on 32-bit
//    shared-window loads.  Any other shape (or a malformed line) takes the exact general paths
//    (cm_parse, cm_parse_serial), so every byte sequence gets the oracle's answer.
//  * CM2: eventType == 1 survivors are ballot-compacted into a per-warp smem ring as SWAR digit
//    words and decoded / aggregated 32 at a time by full warps (dictionary jobId -> index, two
//    RED.64 into the striped pane accumulators).  CM1: per-warp ballot/REDUX reduction per
//    (pane, category) into per-warp smem accumulators, one RED.64 pair per CTA and key.
#include "common.cuh"

#include <mutex>

namespace lms {
namespace {

constexpr int kCmThreads = 128;
constexpr int kWarps = kCmThreads / 32;
constexpr int kCtasPerSm = 5;
constexpr int kCmStages = 2;                                 // per-warp smem ring
constexpr int kChunk = 128;                                  // window chunk per lane
constexpr int kChunks = kCmTile / kChunk;                    // 32 payload chunks per warp tile
static_assert(kChunks == 32, "one payload chunk per lane");
constexpr int kMaskBits = kCmWin;                            // mask bit i <-> stage byte 16 + i
constexpr int kMaskW32 = kMaskBits / 32;                     // 136
constexpr int kPieces = kMaskBits / 16;                      // 272 pieces of 16 B
static_assert(kPieces % 64 == 16, "4 piece pairs + a half row per lane");
constexpr int kSurvCap = 64;                                 // per-warp survivor list
constexpr int kSmemPad = 16;                                 // SWAR loads may read 12 B past a stage

// Pass-1 byte classification, balanced between the ALU pipe (LOP3, SHF: half rate on B200)
// and the FMA pipe (VIADD / IMAD / IDP): per word and class one LOP3 (w & 0x7F..) ^ c, one add,
// one LOP3 for the flags; per 16 B piece and class an IDP.4A chain and one IMAD + SHF.
// Exact byte-equality flags: bit 7 of byte k set iff byte k == c (c < 0x80): the low 7 bits
// equal <=> ((w & 0x7F..) ^ c) + 0x7F.. leaves bit 7 clear, and the byte's own bit 7 is clear.
__device__ __forceinline__ uint32_t lop3_and_xor(uint32_t a, uint32_t b, uint32_t c) {   // (a & b) ^ c
  uint32_t d;
  asm("lop3.b32 %0, %1, %2, %3, 0x6A;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}
__device__ __forceinline__ uint32_t eq_flags(uint32_t w, uint32_t k7f, uint32_t c4) {
  const uint32_t t = lop3_and_xor(w, k7f, c4) + 0x7F7F7F7Fu;
  return ~(t | w) & 0x80808080u;
}
__device__ __forceinline__ uint32_t imad(uint32_t a, uint32_t b, uint32_t c) {   // a * b + c, kept an IMAD
  uint32_t x;
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(x) : "r"(a), "r"(b), "r"(c));
  return x;
}
// 128 * (16-bit mask) of a 16 B piece from four flag words: IDP.4A gathers bytes {0, 0x80}
// to 128 * bits 0..7 per word pair, hi * 256 + lo joins the halves.
__device__ __forceinline__ uint32_t gather16x128(uint32_t f0, uint32_t f1, uint32_t f2, uint32_t f3, uint32_t k256) {
  const uint32_t lo = __dp4a(f1, 0x80402010u, __dp4a(f0, 0x08040201u, 0u));
  const uint32_t hi = __dp4a(f3, 0x80402010u, __dp4a(f2, 0x08040201u, 0u));
  return imad(hi, k256, lo);
}
__device__ __forceinline__ uint32_t sel(bool c, uint32_t a, uint32_t b) {   // c ? a : b, never a branch
  uint32_t d;
  asm("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %1, 0;\n\tselp.b32 %0, %2, %3, p;\n\t}"
      : "=r"(d) : "r"((uint32_t)c), "r"(a), "r"(b));
  return d;
}
// first set bit of a 128-bit chunk mask (chunk base cb), 0xFFFF if none (branch-free)
__device__ __forceinline__ uint32_t first_bit128(uint32_t m0, uint32_t m1, uint32_t m2, uint32_t m3, uint32_t cb) {
  const uint32_t a = sel(m0 != 0u, m0, m1), ka = sel(m0 != 0u, 0u, 32u);
  const uint32_t b = sel(m2 != 0u, m2, m3), kb = sel(m2 != 0u, 64u, 96u);
  const bool lo = (m0 | m1) != 0u;
  const uint32_t w = sel(lo, a, b), k = sel(lo, ka, kb);
  return sel(w != 0u, cb + k + (uint32_t)(__ffs(w) - 1), 0xFFFFu);
}

__device__ __forceinline__ uint4 lds128(uint32_t a) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
  return v;
}
__device__ __forceinline__ uint32_t lds32(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts32(uint32_t a, uint32_t v) {
  asm volatile("st.shared.u32 [%0], %1;" ::"r"(a), "r"(v));
}

struct CmArgs {
  QueryDev q;
  SegTable segs;
  unsigned long long total_tiles;
  uint32_t k7f, k256, k512;          // 0x7F7F7F7F, 256, 512: kernel arguments, so they stay in registers
  uint32_t pane_m, pane_sh;          // pane30: floor(ts / S) = umulhi(ts, pane_m) >> pane_sh
};

// floor(ts / S) for ts < 2^30 (every CM timestamp: <= 9 digits) with a 32-bit magic number:
// k = max(32, 30 + ceil(log2 S)), M = ceil(2^k / S) < 2^31 + 1, shift k - 32.  Exact: ts * M / 2^k
// = ts / S + ts * err / 2^k with 0 <= err < 1, and ts / 2^k < 2^30 / 2^k <= 1 / S, so the error
// never reaches the next multiple of 1 / S.  S = 1: M = 0, the identity (pane_sh = 32 marks it).
__device__ __forceinline__ uint32_t pane30(uint32_t ts, uint32_t m, uint32_t sh) {
  return sh == 32u ? ts : (__umulhi(ts, m) >> sh);
}
void pane30_magic(uint32_t S, uint32_t& m, uint32_t& sh) {
  if (S <= 1) { m = 0; sh = 32; return; }
  uint32_t lg = 0;
  while ((1ull << lg) < S) lg++;
  const uint32_t k = lg + 30 > 32 ? lg + 30 : 32;
  m = (uint32_t)(((1ull << k) + S - 1) / S);
  sh = k - 32;
}

struct TileGeom {
  const uint8_t* seg;
  unsigned long long off;            // tile starts at seg + off
  uint32_t lo, hi;                   // valid smem bytes [lo, hi) (relative to stage start)
  uint32_t payload;                  // tile payload bytes (<= kCmTile)
  bool cont;                         // the next tile continues this segment (its first 256 B = our halo)
};

// A warp's walk over its contiguous tile range: the current tile's segment and offset,
// advanced one tile at a time (the segment changes only at segment ends).  j = tile index in
// the segment; tiles 1..jfull are FULL (left halo, 4096 B payload, whole right halo), the
// common case, whose geometry is constant.
struct TileIter {
  const uint8_t* seg;
  unsigned long long off, nbytes;      // tile start within the segment, segment size
  int si;
  uint32_t j, jend, jfull;             // tile index in the segment, segment tiles, last full tile
  __device__ __forceinline__ void seg_init(const SegTable& s) {
    seg = s.s[si].ptr;
    nbytes = s.s[si].nbytes;
    jend = (uint32_t)(s.tile_prefix[si + 1] - s.tile_prefix[si]);
    jfull = nbytes >= (unsigned long long)kCmWin ? (uint32_t)((nbytes - kCmWin) / kCmTile) : 0u;
  }
  __device__ __forceinline__ void init(const SegTable& s, unsigned long long tile) {
    si = 0;
    while (si + 1 < s.n && tile >= s.tile_prefix[si + 1]) si++;
    seg_init(s);
    j = (uint32_t)(tile - s.tile_prefix[si]);
    off = (unsigned long long)j * kCmTile;
  }
  __device__ __forceinline__ void next(const SegTable& s) {
    off += kCmTile;
    j++;
    while (j >= jend && si + 1 < s.n) { si++; seg_init(s); off = 0; j = 0; }
  }
  __device__ __forceinline__ bool full() const { return j - 1u < jfull; }
  __device__ __forceinline__ TileGeom geom() const {
    TileGeom g;
    g.seg = seg;
    g.off = off;
    if (full()) {
      g.payload = kCmTile;
      g.lo = 0;
      g.hi = kCmStage;
      g.cont = true;
      return g;
    }
    const unsigned long long rem = nbytes - off;
    g.payload = (uint32_t)(rem < (unsigned long long)kCmTile ? rem : kCmTile);
    g.lo = off == 0 ? kCmHaloL : 0;
    g.hi = kCmHaloL + (uint32_t)(rem < (unsigned long long)kCmWin ? rem : kCmWin);
    g.cont = rem > (unsigned long long)kCmTile;
    return g;
  }
};

// mbarrier / bulk copy on precomputed shared-window addresses (no per-tile cvta)
__device__ __forceinline__ void mbar_wait_s(uint32_t bar, uint32_t phase) {
  asm volatile(
      "{\n .reg .pred p;\n CM_WAIT:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra CM_WAIT;\n}" ::"r"(bar), "r"(phase) : "memory");
}
// The input is read once: copies carry an L2 evict-first policy, so a 1.4 GB micro-batch does
// not push the jobId dictionary and the pane accumulators out of the 126 MB L2 (J = 10^6 keys:
// 0.48 -> 0.40 ms per 10M records; J = 10^4: unchanged).
__device__ __forceinline__ void issue_s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
  asm volatile("{\n .reg .b64 pol;\n createpolicy.fractional.L2::evict_first.b64 pol, 1.0;\n"   // read-once input
               " cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], pol;\n}"
               ::"r"(dst), "l"(src), "r"(bytes), "r"(bar) : "memory");
}
struct CmRec {
  uint32_t ts;
  unsigned long long job;
  uint32_t event, cat, cpu_m;
  // fast path, CM2: the jobId and cpu digits as SWAR digit values (byte - '0'); the values are
  // decoded only for survivors, by the drain (cm_job_value / cm_cpu_value)
  uint32_t jw0, jw1, jw2, cw0, cw1;
};
constexpr uint32_t kRawValues = 0xFFFFFFFFu;   // cw1 marker: jw0/jw1 = jobId, cw0 = cpu_m (slow path)

__device__ __forceinline__ bool digits_u32(const uint8_t* b, uint32_t n, uint32_t& v) {
  v = 0;
  for (uint32_t i = 0; i < n; i++) {
    const uint32_t d = (uint32_t)b[i] - 48u;
    if (d > 9u) return false;
    v = v * 10u + d;
  }
  return true;
}
__device__ __forceinline__ bool digits_u64(const uint8_t* b, uint32_t n, unsigned long long& v) {
  v = 0;
  for (uint32_t i = 0; i < n; i++) {
    const uint32_t d = (uint32_t)b[i] - 48u;
    if (d > 9u) return false;
    v = v * 10ull + d;
  }
  return true;
}

// Bytes [p, p+12) of smem as three little-endian words (p arbitrary; reads 16 aligned bytes).
__device__ __forceinline__ void load12(const uint8_t* buf, uint32_t p, uint32_t& d0, uint32_t& d1, uint32_t& d2) {
  const uint32_t* w = reinterpret_cast<const uint32_t*>(buf + (p & ~3u));
  const uint32_t w0 = w[0], w1 = w[1], w2 = w[2], w3 = w[3], sh = (p & 3u) * 8u;
  d0 = __funnelshift_r(w0, w1, sh);
  d1 = __funnelshift_r(w1, w2, sh);
  d2 = __funnelshift_r(w2, w3, sh);
}
// 4 ASCII digits (first character in the low byte) -> value; caller validated the bytes.
__device__ __forceinline__ uint32_t swar4(uint32_t x) {
  x -= 0x30303030u;
  x = x * 10u + (x >> 8);                   // bytes 0, 2: 10*d0+d1, 10*d2+d3
  return (x & 0xFFu) * 100u + ((x >> 16) & 0xFFu);
}
// bit 7 of each byte set iff the byte is NOT an ASCII digit
__device__ __forceinline__ uint32_t nondigit(uint32_t x) {
  const uint32_t t = x ^ 0x30303030u;
  return (((t & 0x7F7F7F7Fu) + 0x76767676u) | t) & 0x80808080u;
}

// Decode + validate given the separator positions (stage-byte offsets): s = record start,
// c[0..9] the first 10 commas (the caller checked there are exactly 12 and the '\n').
__device__ __forceinline__ bool cm_fields(const uint8_t* buf, uint32_t s, const uint32_t (&c)[10], CmRec& r) {
  const uint32_t lts = c[0] - s;
  if (lts < 1 || lts > 9) return false;
  if (!digits_u32(buf + s, lts, r.ts)) return false;
  if (c[1] != c[0] + 1) return false;                      // missing-info field is empty
  const uint32_t lj = c[2] - c[1] - 1;
  if (lj == 10) {                                           // common case: SWAR
    uint32_t d0, d1, d2;
    load12(buf, c[1] + 1, d0, d1, d2);
    if ((nondigit(d0) | nondigit(d1) | (nondigit(d2) & 0x8080u)) != 0) return false;
    const uint32_t hi8 = swar4(d0) * 10000u + swar4(d1);
    const uint32_t lo2 = ((d2 & 0xFFu) - 48u) * 10u + (((d2 >> 8) & 0xFFu) - 48u);
    r.job = (unsigned long long)hi8 * 100ull + lo2;
  } else {
    if (lj < 1 || lj > 19) return false;
    if (!digits_u64(buf + c[1] + 1, lj, r.job)) return false;
  }
  if (c[5] != c[4] + 2 || c[7] != c[6] + 2 || c[9] != c[8] + 9) return false;
  r.event = (uint32_t)buf[c[4] + 1] - 48u;
  r.cat = (uint32_t)buf[c[6] + 1] - 48u;
  if (r.event > 9u || r.cat > 9u) return false;
  uint32_t d0, d1, d2;                                      // cpu = D.DDDDDD (8 bytes)
  load12(buf, c[8] + 1, d0, d1, d2);
  const uint32_t dot = (d0 >> 8) & 0xFFu;
  const uint32_t nd = (nondigit(d0) & 0x80800080u) | nondigit(d1);   // bytes 0, 2..7 digits
  if (dot != '.' || nd) return false;
  const uint32_t ip = (d0 & 0xFFu) - 48u;
  // fraction digits: d0 bytes 2,3 ; d1 bytes 0..3
  const uint32_t f2 = (((d0 >> 16) & 0xFFu) - 48u) * 10u + (((d0 >> 24) & 0xFFu) - 48u);
  r.cpu_m = ip * 1000000u + f2 * 10000u + swar4(d1);
  (void)d2;
  return true;
}

// Exact byte-serial path: any line the fast path does not cover (short / long / malformed).
__device__ __forceinline__ bool cm_parse_serial(const uint8_t* buf, uint32_t s, uint32_t limit, CmRec& r) {
  uint32_t c[10];
  uint32_t nc = 0;
  const uint32_t stop = min(limit, s + kCmMaxLine + 1);
  for (uint32_t i = s; i < stop; i++) {
    const uint8_t b = buf[i];
    if (b == '\n') {
      if (nc != 12) return false;
      return cm_fields(buf, s, c, r);
    }
    if (b == ',') {
      if (nc >= 12) return false;
      if (nc < 10) c[nc] = i;
      nc++;
    }
  }
  return false;   // no '\n' within 256 bytes or before the segment end
}

// ---- 32-bit mask helpers (the '\n' / ',' masks are read as 32-bit words: bit i of the
// window <-> word i >> 5, bit i & 31)
__device__ __forceinline__ uint32_t lsb32(uint32_t x) { return (uint32_t)__ffs(x) - 1u; }   // x != 0
__device__ __forceinline__ uint32_t msb32(uint32_t x) {                                   // x != 0
  uint32_t r;
  asm("bfind.u32 %0, %1;" : "=r"(r) : "r"(x));
  return r;
}
// low n bits set, n in [0, 32] (PTX shl clamps: 1 << 32 == 0)
__device__ __forceinline__ uint32_t low_bits(uint32_t n) {
  uint32_t r;
  asm("{\n\t.reg .b32 t;\n\tshl.b32 t, 1, %1;\n\tsub.u32 %0, t, 1;\n\t}" : "=r"(r) : "r"(n));
  return r;
}
__device__ __forceinline__ uint32_t clamp32(int n) { return (uint32_t)min(max(n, 0), 32); }

// Pop the lowest set bit of the 128-bit chunk mask s0..s3 into b (chunk-relative).
__device__ __forceinline__ bool pop_lowest(uint32_t& s0, uint32_t& s1, uint32_t& s2, uint32_t& s3, uint32_t& b) {
  const uint32_t w = s0 ? s0 : (s1 ? s1 : (s2 ? s2 : s3));
  if (!w) return false;
  const uint32_t k = s0 ? 0u : (s1 ? 1u : (s2 ? 2u : 3u));
  b = 32u * k + lsb32(w);
  const uint32_t wc = w & (w - 1u);
  s0 = k == 0 ? wc : s0;
  s1 = k == 1 ? wc : s1;
  s2 = k == 2 ? wc : s2;
  s3 = k == 3 ? wc : s3;
  return true;
}

// Parse the record starting at mask bit sb whose '\n' is at mask bit e (e > sb).
// Returns 1 valid, 0 malformed, 2 undecided (the caller runs the exact byte-serial path).
// Mask path (64 <= L = e - sb <= 191): the comma count of [sb, e) from a 192-bit window at sb
// (must be 12: 13 fields); commas 0..5 are the 6 lowest bits of its first 64 bits, commas
// 6..11 the 6 highest bits of the 64-bit window ending at e.
__device__ __forceinline__ int cm_parse(const uint8_t* buf, const uint32_t* cm32, uint32_t sb, uint32_t e,
                                        uint32_t hi_bits, CmRec& r) {
  const uint32_t S = kCmHaloL + sb;
  const uint32_t L = e - sb;
  if (L - 64u > 127u) return 2;
  const uint32_t* w = cm32 + (sb >> 5);
  const uint32_t sh = sb & 31u;
  const uint32_t v0 = w[0], v1 = w[1], v2 = w[2], v3 = w[3], v4 = w[4], v5 = w[5], v6 = w[6];
  uint32_t h0 = __funnelshift_r(v0, v1, sh), h1 = __funnelshift_r(v1, v2, sh);
  const uint32_t x2 = __funnelshift_r(v2, v3, sh) & low_bits(clamp32((int)L - 64));
  const uint32_t x3 = __funnelshift_r(v3, v4, sh) & low_bits(clamp32((int)L - 96));
  const uint32_t x4 = __funnelshift_r(v4, v5, sh) & low_bits(clamp32((int)L - 128));
  const uint32_t x5 = __funnelshift_r(v5, v6, sh) & low_bits(clamp32((int)L - 160));
  const uint32_t nh = __popc(h0) + __popc(h1);
  if (nh + __popc(x2) + __popc(x3) + __popc(x4) + __popc(x5) != 12u) return 0;   // not 13 fields
  // tail window [e - 64, e)
  const uint32_t tp = e - 64u;
  const uint32_t* u = cm32 + (tp >> 5);
  const uint32_t tsh = tp & 31u, u0 = u[0], u1 = u[1], u2 = u[2];
  uint32_t t0 = __funnelshift_r(u0, u1, tsh), t1 = __funnelshift_r(u1, u2, tsh);
  if (nh < 6u || __popc(t0) + __popc(t1) < 6u) return 2;
  uint32_t c[10];
  // ---- head: commas 0..5 = the 6 lowest bits of h1:h0.  c0 ends ts (1..9 digits), c1 = c0 + 1
  // (empty field 1): anything else is malformed.  Usual shape: a 10-digit jobId, so c2 =
  // c0 + 12 is read off the mask; taskIndex / machineId are free-form: two pops give c3, c4.
  const uint32_t o0 = lsb32(h0 | 0x80000000u);               // h0 == 0: ts > 31 bytes
  if (o0 - 1u > 8u || ((h0 >> (o0 + 1u)) & 1u) == 0) return 0;
  const uint32_t j0 = __funnelshift_r(h0, h1, o0 + 2u), j1 = h1 >> (o0 + 2u);   // from the jobId
  if ((j0 & 0x7FFu) == 0x400u) {
    c[0] = S + o0;
    c[1] = S + o0 + 1u;
    c[2] = S + o0 + 12u;
    uint32_t r0 = __funnelshift_r(j0, j1, 11u), r1 = j1 >> 11;   // bits after c2
    const uint32_t base = S + o0 + 13u;
#pragma unroll
    for (int k = 3; k < 5; k++) {
      const bool l = r0 != 0;
      const uint32_t t = l ? r0 : r1;
      const uint32_t bit = lsb32(t);
      c[k] = base + bit + (l ? 0u : 32u);                    // r1 holds bits 32.. of r
      const uint32_t tc = t & (t - 1u);
      r0 = l ? tc : r0;
      r1 = l ? r1 : tc;
    }
    // eventType must be 1 char: the next comma (c5) sits at c4 + 2
    c[5] = base + (r0 ? lsb32(r0) : 32u + lsb32(r1));
    if (c[5] != c[4] + 2u) return 0;
  } else {
#pragma unroll
    for (int k = 0; k < 6; k++) {
      const bool l = h0 != 0;
      const uint32_t t = l ? h0 : h1;
      const uint32_t bit = lsb32(t);
      c[k] = S + bit + (l ? 0u : 32u);
      const uint32_t tc = t & (t - 1u);
      h0 = l ? tc : h0;
      h1 = l ? h1 : tc;
    }
  }
  // ---- tail: commas 6..11 = the 6 highest bits of the window [e-64, e).  Usual shape:
  // cpu, ram, disk 8 chars and a 1-char constraint, i.e. commas exactly at e-29, e-20, e-11,
  // e-2 in [e-30, e); then c7 = the next comma below and c6 = c7 - 2 (1-char category).
  const uint32_t T0 = kCmHaloL + tp;
  if ((t1 >> 2) == 0x10080402u) {
    c[8] = T0 + 35u;
    c[9] = T0 + 44u;
    const uint32_t l7 = t1 & 7u;
    const uint32_t q7 = l7 ? 32u + msb32(l7) : msb32(t0);     // window bit of c7 (t0 != 0)
    c[7] = T0 + q7;
    // the comma before c7 must be at c7 - 2: bit q7-1 clear, bit q7-2 set
    const uint32_t w2 = __funnelshift_rc(t0, t1, q7 - 2u) & 3u;   // window bits q7-2, q7-1
    if (q7 < 2u || w2 != 1u) return 0;
    c[6] = c[7] - 2u;
  } else {
#pragma unroll
    for (int k = 11; k >= 6; k--) {
      const bool h = t1 != 0;
      const uint32_t t = h ? t1 : t0;
      const uint32_t bit = msb32(t);
      if (k < 10) c[k] = T0 + bit + (h ? 32u : 0u);
      const uint32_t tc = t ^ (1u << bit);
      t1 = h ? tc : t1;
      t0 = h ? t0 : tc;
    }
  }
  return cm_fields(buf, S, c, r) ? 1 : 0;
}

// Shared-window (32-bit address) forms for the fast path: no 64-bit generic address math.
__device__ __forceinline__ uint32_t lds_u8(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
// Bytes [a, a+8) / [a, a+12) of shared memory at any alignment (reads the aligned words).
__device__ __forceinline__ void lds8u(uint32_t a, uint32_t& d0, uint32_t& d1) {
  const uint32_t b = a & ~3u, sh = (a & 3u) * 8u;
  const uint32_t w0 = lds32(b), w1 = lds32(b + 4), w2 = lds32(b + 8);
  d0 = __funnelshift_r(w0, w1, sh);
  d1 = __funnelshift_r(w1, w2, sh);
}
__device__ __forceinline__ void lds12u(uint32_t a, uint32_t& d0, uint32_t& d1, uint32_t& d2) {
  const uint32_t b = a & ~3u, sh = (a & 3u) * 8u;
  const uint32_t w0 = lds32(b), w1 = lds32(b + 4), w2 = lds32(b + 8), w3 = lds32(b + 12);
  d0 = __funnelshift_r(w0, w1, sh);
  d1 = __funnelshift_r(w1, w2, sh);
  d2 = __funnelshift_r(w2, w3, sh);
}

// Bytes [p, p+8) of smem as two little-endian words (p arbitrary; reads 12 aligned bytes).
__device__ __forceinline__ void load8(const uint8_t* buf, uint32_t p, uint32_t& d0, uint32_t& d1) {
  const uint32_t* w = reinterpret_cast<const uint32_t*>(buf + (p & ~3u));
  const uint32_t w0 = w[0], w1 = w[1], w2 = w[2], sh = (p & 3u) * 8u;
  d0 = __funnelshift_r(w0, w1, sh);
  d1 = __funnelshift_r(w1, w2, sh);
}

// SWAR digit helpers on d = x - 0x30303030 (x: 4 ASCII bytes, first character in the low byte).
// dbad(d): bit 7 of some byte is set iff some byte of x is not an ASCII digit.  Proof: let k be
// the lowest non-digit byte (no borrow reaches it); x_k < '0' wraps d_k to >= 0xD0, and
// x_k > '9' gives d_k >= 0x0A, so d_k has bit 7 set or d_k + 0x76 does (the digit bytes below
// k add at most 0x7F: no carry into byte k).  All digits: d_k <= 9, d_k + 0x76 <= 0x7F.
__device__ __forceinline__ uint32_t dbad(uint32_t d) { return d | (d + 0x76767676u); }
// value of 4 digit values (first = most significant): pairs 10*d0+d1, 10*d2+d3 land in bytes
// 1 and 3 of d * 0xA01 (each <= 99: no carries), PRMT moves them to bytes 0 and 2, and
// (p * (100 << 16 | 1)) >> 16 = 100 * pair0 + pair1.
__device__ __forceinline__ uint32_t swar4d(uint32_t d) {
  const uint32_t p = __byte_perm(d * 0xA01u, 0u, 0x4341u);
  return (p * 0x640001u) >> 16;
}

// Straight-line (branch-free) decode of a record of the USUAL shape: 128 <= L <= 191, exactly
// 12 commas, ts of 1..8 digits, empty field 1, a 10-digit jobId, a 1-character eventType,
// then (user free-form) a 1-character category, a 1..2-character priority and, at the tail,
// cpu, ram, disk (8 characters each) and a 1-character constraint.  Returns true iff the
// record has that shape AND is valid under reading R1 (then r holds its fields); false means
// "not decided here": the caller re-parses the record with the exact general path (cm_parse),
// so the fast path never rejects anything itself.  sb / e: mask bits of the record start and
// of its '\n' (sb <= 4096).  Every smem address stays inside the stage (see `ec`), so that
// predicated-off garbage positions cannot fault.
// The exact general path for a record the fast path did not accept (other field shapes,
// malformed lines), out of line: it is rare, and kept out of the hot loop's instruction
// footprint.  Values come back in registers (no address of the caller's record escapes).
struct CmSlow {
  uint32_t ok, ts, event, cat, cpu_m, job_lo, job_hi;
};
__device__ __noinline__ CmSlow cm_slow(const uint8_t* buf, const uint32_t* cm32, uint32_t sb, uint32_t e,
                                       uint32_t hi_bits) {
  CmRec r{};
  const int st = e == 0xFFFFu ? 2 : cm_parse(buf, cm32, sb, e, hi_bits, r);
  const bool ok = st == 2 ? cm_parse_serial(buf, kCmHaloL + sb, hi_bits + kCmHaloL, r) : st != 0;
  CmSlow o;
  o.ok = ok ? 1u : 0u;
  o.ts = r.ts; o.event = r.event; o.cat = r.cat; o.cpu_m = r.cpu_m;
  o.job_lo = (uint32_t)r.job; o.job_hi = (uint32_t)(r.job >> 32);
  return o;
}

template <bool kLazy>
// buf_s / cm_s: shared-window addresses of the stage and of the warp's comma mask words.
__device__ __forceinline__ bool cm_fast(uint32_t buf_s, uint32_t cm_s, uint32_t sb, uint32_t e, CmRec& r) {
  const uint32_t S = kCmHaloL + sb;
  const uint32_t L = e - sb;
  bool ok = L - 128u <= 63u;
  // ---- comma windows: head [sb, sb+64), middle [sb+64, e-64), tail [e-64, e)
  const uint32_t wa = cm_s + 4u * (sb >> 5);
  const uint32_t sh = sb & 31u;
  const uint32_t v0 = lds32(wa), v1 = lds32(wa + 4), v2 = lds32(wa + 8), v3 = lds32(wa + 12), v4 = lds32(wa + 16);
  const uint32_t h0 = __funnelshift_r(v0, v1, sh), h1 = __funnelshift_r(v1, v2, sh);
  const unsigned long long mid = (((unsigned long long)__funnelshift_r(v3, v4, sh) << 32) | __funnelshift_r(v2, v3, sh)) &
                                 ((1ull << min(L - 128u, 63u)) - 1ull);          // bits [sb+64, e-64)
  // e clamped into the window for addressing only (e = 0xFFFF: no '\n' in reach; L above
  // already rejects it): with S <= 16 + 4096 and o0, a4, q7 < 35 every load below stays
  // inside the stage, so no address needs its own clamp
  const uint32_t ec = min(max(e, 64u), (uint32_t)kMaskBits - 1u);
  const uint32_t tp = ec - 64u;
  const uint32_t ua = cm_s + 4u * (tp >> 5);
  const uint32_t tsh = tp & 31u, u0 = lds32(ua), u1 = lds32(ua + 4), u2 = lds32(ua + 8);
  const uint32_t t0 = __funnelshift_r(u0, u1, tsh), t1 = __funnelshift_r(u1, u2, tsh);
  // ---- head: c0 = sb + o0 ends ts (1..8 digits); c1 = c0 + 1 (empty field 1); c2 = c0 + 12
  // (10-digit jobId); then taskIndex, machineId free-form: c4 = the 2nd comma after c2, and
  // eventType is 1 character: the next comma (c5) is at c4 + 2.
  const uint32_t o0 = lsb32(h0 | 0x80000000u);
  ok &= o0 - 1u <= 7u;
  const uint32_t jw = __funnelshift_r(h0, h1, o0 + 1u);           // bit 0 <-> c1
  ok &= (jw & 0xFFFu) == 0x801u;
  const uint32_t rr = __funnelshift_r(h0, h1, o0 + 13u);          // bits after c2
  const uint32_t x = rr & (rr - 1u);                              // c3 cleared
  const uint32_t a4 = lsb32(x | 0x80000000u);                     // c4 = c2 + 1 + a4
  ok &= x != 0u && a4 <= 29u && ((x >> a4) & 7u) == 5u;
  // ---- exactly 12 commas: the head checks pin c0..c5 as the only commas in [sb, c5] and the
  // tail checks below pin c6..c11 as the only ones in window bits [30, 64) = [e-34, e), so the
  // record has 13 fields iff no comma lies after c5 in the head window, none in the middle
  // [sb+64, e-64), and none in tail bits [0, 30) (c5 <= sb + 52 < the tail's start: L >= 128)
  const unsigned long long head = ((unsigned long long)h1 << 32) | h0;
  const unsigned long long after_c5 = head >> ((o0 + 16u + a4) & 63u);
  ok &= ((after_c5 | mid) == 0ull) & ((t0 & 0x3FFFFFFFu) == 0u);
  // ---- tail, window [e-64, e): commas exactly at e-29, e-20, e-11, e-2 within [e-30, e)
  // (cpu, ram, disk 8 chars, constraint 1 char); c7 (priority end) at e-31 or e-32 and
  // c6 = c7 - 2 (1-char category): window bits 30..34 = 0b01010 or 0b00101.
  ok &= (t1 >> 2) == 0x10080402u;
  const uint32_t pc = __funnelshift_r(t0, t1, 30u) & 0x1Fu;
  ok &= pc == 0x0Au || pc == 0x05u;
  const uint32_t cat_at = kCmHaloL + ec - (pc == 0x0Au ? 32u : 33u);  // c6 + 1
  // ---- fields (digit checks accumulate into bad; bit 7 of a byte = not a digit)
  // ts: bytes [S, S + 8) hold its o0 digits, then ','.  '0' is subtracted from all 8 bytes as one
  // 64-bit subtraction (borrows only run toward later bytes, i.e. past the digits; a non-digit
  // byte among the digits is caught below), then the digit values are shifted to the top of the
  // word: the bytes after them fall off, zero bytes (leading zeros) come in below.
  uint32_t a0, a1;
  lds8u(buf_s + S, a0, a1);
  const unsigned long long ta = (((unsigned long long)a1 << 32) | a0) - 0x3030303030303030ull;
  const unsigned long long tv = ta << (8u * ((8u - o0) & 7u));
  const uint32_t da0 = (uint32_t)tv, da1 = (uint32_t)(tv >> 32);
  uint32_t bad = dbad(da0) | dbad(da1);
  r.ts = swar4d(da0) * 10000u + swar4d(da1);
  // jobId: 10 digits at c1 + 1 = S + o0 + 2
  uint32_t d0, d1, d2;
  lds12u(buf_s + S + o0 + 2u, d0, d1, d2);
  d0 -= 0x30303030u;
  d1 -= 0x30303030u;
  d2 -= 0x30303030u;
  bad |= dbad(d0) | dbad(d1) | (dbad(d2) & 0x8080u);
  r.jw0 = d0;
  r.jw1 = d1;
  r.jw2 = d2;
  // eventType at c4 + 1 = S + o0 + 14 + a4; category at c6 + 1
  r.event = lds_u8(buf_s + S + o0 + 14u + a4) - 48u;
  r.cat = lds_u8(buf_s + cat_at) - 48u;
  ok &= r.event <= 9u && r.cat <= 9u;
  // cpu = D.DDDDDD at c8 + 1 = e - 28: the '.' is swapped for '0' for the digit check and
  // SWAR value (D0DD DDDD), and the integer digit's weight is fixed up (10^7 -> 10^6)
  uint32_t p0, p1;
  lds8u(buf_s + kCmHaloL + ec - 28u, p0, p1);
  ok &= ((p0 >> 8) & 0xFFu) == '.';
  const uint32_t dp0 = (p0 ^ 0x1E00u) - 0x30303030u, dp1 = p1 - 0x30303030u;
  bad |= dbad(dp0) | dbad(dp1);
  if (kLazy) {
    r.cw0 = dp0;
    r.cw1 = dp1;
  } else {
    r.cpu_m = swar4d(dp0) * 10000u + swar4d(dp1) - 9000000u * (dp0 & 0xFFu);
  }
  return ok && (bad & 0x80808080u) == 0u;
}

// Values of the digit words cm_fast kept (jobId: 10 digits in jw0..jw2; cpu: D0DDDDDD in cw0, cw1
// with the integer digit's weight fixed up 10^7 -> 10^6), or the slow path's values (kRawValues).
__device__ __forceinline__ unsigned long long cm_job_value(uint32_t jw0, uint32_t jw1, uint32_t jw2, uint32_t cw1) {
  const uint32_t lo2 = __byte_perm(jw2 * 0xA01u, 0u, 0x4441u);     // 10 * d2_0 + d2_1
  const unsigned long long v = (unsigned long long)(swar4d(jw0) * 10000u + swar4d(jw1)) * 100ull + lo2;
  return cw1 == kRawValues ? ((unsigned long long)jw1 << 32 | jw0) : v;
}
__device__ __forceinline__ uint32_t cm_cpu_value(uint32_t cw0, uint32_t cw1) {
  const uint32_t v = swar4d(cw0) * 10000u + swar4d(cw1) - 9000000u * (cw0 & 0xFFu);
  return cw1 == kRawValues ? cw0 : v;
}

// Tile geometry, packed into one word when the tile's copy is issued (two tiles before it is
// consumed): payload bytes [0, 13), valid mask bits (stage bytes [16, 16 + hi_bits)) [13, 26),
// segment start (left halo invalid) bit 26, the next tile continues the segment bit 27.
constexpr uint32_t kGeoFull = (uint32_t)kCmTile | ((uint32_t)kCmWin << 13) | (1u << 27);
__device__ __forceinline__ uint32_t geo_payload(uint32_t g) { return g & 0x1FFFu; }
__device__ __forceinline__ uint32_t geo_hibits(uint32_t g) { return (g >> 13) & 0x1FFFu; }
__device__ __forceinline__ bool geo_start(uint32_t g) { return (g >> 26) & 1u; }
__device__ __forceinline__ bool geo_cont(uint32_t g) { return (g >> 27) & 1u; }

// Issue the copy of the producer iterator's tile into stage `dst` (shared-window address) and
// return its packed geometry.  Full tiles: one constant-size copy.  Segment heads / tails: the
// 16 B-multiple part by the TMA engine, the < 16 B remainder by lane 0 right here (the stage is
// free, the bytes are disjoint from the bulk copy's, and the warp synchronises before it reads
// the stage again).
__device__ __forceinline__ uint32_t cm_issue(const TileIter& it, uint32_t dst, uint32_t bar, int lane) {
  if (it.full()) {
    if (lane == 0) issue_s(dst, it.seg + it.off - kCmHaloL, kCmStage, bar);
    return kGeoFull;
  }
  const TileGeom g = it.geom();
  const uint32_t bulk = (g.hi - g.lo) & ~15u;
  if (lane == 0) {
    if (bulk) issue_s(dst + g.lo, g.seg + g.off - kCmHaloL + g.lo, bulk, bar);
    else asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(0u) : "memory");
    for (uint32_t i = g.lo + bulk; i < g.hi; i++)
      asm volatile("st.shared.u8 [%0], %1;" ::"r"(dst + i), "r"((uint32_t)g.seg[g.off - kCmHaloL + i]));
  }
  return g.payload | ((g.hi - kCmHaloL) << 13) | ((g.lo != 0 ? 1u : 0u) << 26) | ((g.cont ? 1u : 0u) << 27);
}

template <int KIND>
__global__ void __launch_bounds__(kCmThreads, kCtasPerSm) k_cm_agg(const CmArgs a) {
  constexpr bool kCM2 = (KIND == kCM2S);
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(8) uint64_t full[kWarps][kCmStages];
  __shared__ unsigned long long slot_tag[2];
  // per-warp '\n' / ',' masks of the warp's current window (+ zero words for reads past it)
  __shared__ __align__(16) uint32_t nlm[kWarps][kMaskW32 + 8], cmm[kWarps][kMaskW32 + 8];
  // (static + dynamic shared memory must stay <= 233472 / 5 - 1024 B per CTA: 5 CTAs per SM)
  // CM2: per-warp survivor rings (jobId / cpu digit words, pane); CM1: per-warp accumulators
  constexpr int kSv = kCM2 ? kWarps : 1;
  // {jobId digits 0-3, 4-7 (+ 8, 9 in the high nibbles of bytes 0, 1 of the first word), cpu
  // words}: one 16 B store / load per survivor
  __shared__ uint4 sv_e[kSv][kSurvCap];
  __shared__ uint32_t sv_p[kSv][kSurvCap];
  __shared__ unsigned long long w_sum[kCM2 ? 1 : kWarps][kCM2 ? 1 : 2][kCM2 ? 1 : 10];
  __shared__ unsigned long long w_cnt[kCM2 ? 1 : kWarps][kCM2 ? 1 : 2][kCM2 ? 1 : 10];
  static_assert(sizeof(nlm) >= 1280, "flush_counters scratch");

  const QueryDev& q = a.q;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // every warp walks its own contiguous range of warp tiles: no CTA barrier in the loop
  const unsigned long long T = a.total_tiles, GW = (unsigned long long)gridDim.x * kWarps;
  const unsigned long long gw = (unsigned long long)blockIdx.x * kWarps + warp;
  const unsigned long long t0 = T * gw / GW, t1 = T * (gw + 1) / GW;
  uint8_t* const wsmem = smem + warp * (kCmStages * kCmStage);
  uint32_t* const nl32 = nlm[warp];
  uint32_t* const cm32 = cmm[warp];

  if (!kCM2)
    for (int i = tid; i < (int)(sizeof(w_sum) / 8); i += blockDim.x) {
      (&w_sum[0][0][0])[i] = 0;
      (&w_cnt[0][0][0])[i] = 0;
    }
  if (tid < 2) slot_tag[tid] = kEmpty64;
  if (lane < 8) { nl32[kMaskW32 + lane] = 0; cm32[kMaskW32 + lane] = 0; }   // reads past the end
  if (lane == 0) {
    for (int s = 0; s < kCmStages; s++) mbar_init(&full[warp][s], 1);
    mbar_fence_init();
  }
  __syncthreads();
  const uint32_t ntiles = (uint32_t)(t1 - t0);
  const uint32_t nl_s = smem_addr(nl32), cm_s = smem_addr(cm32);
  const uint32_t full_s = smem_addr(&full[warp][0]), stage_s = smem_addr(wsmem);
  TileIter iss;                                // producer: the next tile to issue
  iss.init(a.segs, t0);
  uint32_t geo0 = 0, geo1 = 0;                 // packed geometry of the tiles in stages 0 / 1
  if (ntiles > 0) { geo0 = cm_issue(iss, stage_s, full_s, lane); iss.next(a.segs); }
  if (ntiles > 1) { geo1 = cm_issue(iss, stage_s + kCmStage, full_s + 8u, lane); iss.next(a.segs); }

  const unsigned long long wm_prev = q.state->wm_prev;
  const uint32_t k7f = a.k7f, k256 = a.k256, k512 = a.k512;    // runtime constants (see eq_flags)
  const uint32_t wm32 = (uint32_t)min(wm_prev, 0xFFFFFFFFull);  // late iff ts + 1 < wm_prev (ts < 1e9)
  uint32_t n_rec = 0, n_bad = 0, n_late = 0, n_ovf = 0, ts_min = kEmpty32, ts_max1 = 0;
  uint32_t c_pane = kEmpty32, c_slot = 0, c_gslot = kFail32;   // cached slots of the last pane seen
  unsigned long long* c_sum = nullptr;                          // CM2: the cached pane's stripe
  unsigned long long* c_cnt = nullptr;
  uint32_t sv_h = 0, sv_n = 0;                                  // CM2 survivor ring: head, entries

  // CM2: decode and aggregate ring entries [sv_h, sv_h + n) with the warp's lanes
  auto drain = [&](uint32_t n) {
    __syncwarp();
    if ((uint32_t)lane < n) {
      const uint32_t i = (sv_h + lane) & (kSurvCap - 1);
      const uint32_t w = kCM2 ? warp : 0;
      const uint32_t pp = sv_p[w][i];
      const uint4 ev = sv_e[w][i];
      const bool raw = ev.w == kRawValues;
      const unsigned long long job = cm_job_value(raw ? ev.x : (ev.x & 0x0F0F0F0Fu), ev.y, (ev.x >> 4) & 0x0F0Fu, ev.w);
      const uint32_t m = cm_cpu_value(ev.z, ev.w);
      if (pp != c_pane) {
        c_pane = pp;
        c_gslot = claim_slot(q, pp);
        const size_t base = ((size_t)c_gslot * q.stripes + (blockIdx.x & (q.stripes - 1u))) * q.K;
        c_sum = q.acc_sum + base;
        c_cnt = q.acc_cnt + base;
      }
      const uint32_t idx = c_gslot != kFail32 ? dict_get(q.dict, job, q.state) : kEmpty32;
      if (idx == kEmpty32) n_ovf++;
      else {
        atomicAdd(c_sum + idx, (unsigned long long)m);
        atomicAdd(c_cnt + idx, 1ull);
      }
    }
    sv_h = (sv_h + n) & (kSurvCap - 1);
    __syncwarp();
  };

  bool fresh = true;              // window bits [0, 256) not inherited from the previous tile
  uint32_t carry_nl = 0;          // a record starts at the tile's payload byte 0 (the previous
                                  // tile's last payload byte is a '\n', or a segment start)
  for (uint32_t it = 0; it < ntiles; it++) {
    const uint32_t s = it & 1u;                                 // kCmStages == 2
    const uint32_t ph = (it >> 1) & 1u;
    const uint32_t geo = s ? geo1 : geo0;
    const uint32_t st_s = stage_s + s * (uint32_t)kCmStage;    // stage base (shared window)
    const uint8_t* buf = wsmem + s * kCmStage;
    mbar_wait_s(full_s + 8u * s, ph);                           // every lane: TMA bytes visible
    __syncwarp();                                               // lane 0's remainder bytes (tail tiles)
    const uint32_t hi_bits = geo_hibits(geo);                   // mask bits beyond are invalid
    // ---- Pass 1: exact '\n' / ',' masks, one 32-bit mask word (32 B) per lane per step.
    // Window bits [0, 256) are the previous tile's halo masks when the tile continues the
    // segment (carried below), so a tile classifies 4096 new bytes: 4 words per lane.
    const uint32_t buf_s = st_s + kCmHaloL;
    auto mword = [&](int wi) {
      const uint4 va = lds128(buf_s + 32 * wi), vb = lds128(buf_s + 32 * wi + 16);
      const uint32_t na = gather16x128(eq_flags(va.x, k7f, 0x0A0A0A0Au), eq_flags(va.y, k7f, 0x0A0A0A0Au),
                                       eq_flags(va.z, k7f, 0x0A0A0A0Au), eq_flags(va.w, k7f, 0x0A0A0A0Au), k256);
      const uint32_t nb = gather16x128(eq_flags(vb.x, k7f, 0x0A0A0A0Au), eq_flags(vb.y, k7f, 0x0A0A0A0Au),
                                       eq_flags(vb.z, k7f, 0x0A0A0A0Au), eq_flags(vb.w, k7f, 0x0A0A0A0Au), k256);
      const uint32_t ca = gather16x128(eq_flags(va.x, k7f, 0x2C2C2C2Cu), eq_flags(va.y, k7f, 0x2C2C2C2Cu),
                                       eq_flags(va.z, k7f, 0x2C2C2C2Cu), eq_flags(va.w, k7f, 0x2C2C2C2Cu), k256);
      const uint32_t cb2 = gather16x128(eq_flags(vb.x, k7f, 0x2C2C2C2Cu), eq_flags(vb.y, k7f, 0x2C2C2C2Cu),
                                        eq_flags(vb.z, k7f, 0x2C2C2C2Cu), eq_flags(vb.w, k7f, 0x2C2C2C2Cu), k256);
      sts32(nl_s + 4 * wi, imad(nb, k512, na >> 7));       // (128 mb) * 512 = mb << 16
      sts32(cm_s + 4 * wi, imad(cb2, k512, ca >> 7));
    };
#pragma unroll
    for (int k = 0; k < 4; k++) mword(8 + lane + 32 * k);
    fresh = fresh || geo_start(geo);
    if (fresh) {                                 // (warp-uniform)
      if (lane < 8) mword(lane);
      // a record starts at payload byte 0 iff the tile starts its segment or follows a '\n'
      carry_nl = geo_start(geo) || buf[kCmHaloL - 1] == '\n';
    }
    __syncwarp();
    if (hi_bits < (uint32_t)kMaskBits) {        // segment tail (warp-uniform): clear stale bits
      for (uint32_t wi = lane; wi < (uint32_t)kMaskW32; wi += 32) {
        const uint32_t keep = low_bits(clamp32((int)hi_bits - 32 * (int)wi));
        nl32[wi] &= keep;
        cm32[wi] &= keep;
      }
      __syncwarp();
    }
    // ---- Pass 2: lane l owns payload chunk l (128 B, mask words 4l..4l+3).  A record starts
    // after a '\n' (or at a segment start) and belongs to the chunk holding its first byte;
    // its '\n' is the first newline of chunk l+1, else of chunk l+2 (else the line is longer
    // than 256 B: serial path).  Chunks 32, 33 are the right halo.
    const uint32_t cb = lane * kChunk;
    const uint4 nw = lds128(nl_s + 16 * lane);
    const uint4 nx = lds128(nl_s + 16 * (lane + 2));
    const uint32_t f_mine = first_bit128(nw.x, nw.y, nw.z, nw.w, cb);           // my first '\n'
    const uint32_t f2 = first_bit128(nx.x, nx.y, nx.z, nx.w, cb + 2 * kChunk);  // chunk l+2's
    const uint32_t f1s = __shfl_down_sync(0xffffffffu, f_mine, 1);
    const uint32_t f32 = __shfl_sync(0xffffffffu, f2, 30);      // chunk 32
    const uint32_t f1 = sel(lane == 31, f32, f1s);
    const uint32_t e_after = sel(f1 != 0xFFFFu, f1, f2);       // first '\n' past my chunk
    // Records are owned by the '\n' before them: lane l takes the record after each '\n' of
    // its chunk (if it starts inside the payload); lane 0 also takes the record at payload byte
    // 0 when the tile starts a segment or the byte before it is a '\n'.
    const bool start0 = lane == 0 && carry_nl != 0;
    carry_nl = __shfl_sync(0xffffffffu, nw.w, 31) >> 31;       // last payload byte, for the next tile
    const uint32_t pay = geo_payload(geo);
    uint32_t n0 = nw.x, n1 = nw.y, n2 = nw.z, n3 = nw.w;             // unconsumed newlines (generic lanes)
    const uint32_t cnt_nl = __popc(n0) + __popc(n1) + __popc(n2) + __popc(n3);
    // round 0 serves the usual lane: at most one '\n' in the chunk, no record at byte 0 (records
    // are >= 130 B > a chunk); every other lane walks its records in the generic rounds 1, 2, ...
    const bool simple = cnt_nl <= 1u && !start0;
    bool have = simple && cnt_nl == 1u && f_mine + 1u < pay;
    uint32_t sb = f_mine + 1u, e = e_after;
    bool more = !simple, pend0 = start0;
    // ---- Pass 3: decode my records; aggregate (one record per lane per round)
    while (true) {
      CmRec r;
      bool surv = false;
      n_rec += have ? 1u : 0u;
      sb = sel(have, sb, 0u);
      // usual-shape records: branch-free fast path; anything else: the exact general path
      const bool fast = cm_fast<kCM2>(st_s, cm_s, sb, e, r) & have;
      const bool slow = have & !fast;
      bool ok = fast;
      if (__any_sync(0xffffffffu, slow)) {
        if (slow) {
          const CmSlow o = cm_slow(buf, cm32, sb, e, hi_bits);
          ok = o.ok != 0;
          r.ts = o.ts; r.event = o.event; r.cat = o.cat; r.cpu_m = o.cpu_m;
          if (kCM2) {                  // values, not digit words (cm_job_value / cm_cpu_value)
            r.jw0 = o.job_lo;
            r.jw1 = o.job_hi;
            r.jw2 = 0;
            r.cw0 = o.cpu_m;
            r.cw1 = kRawValues;
          }
        }
      }
      {   // drop malformed (counted) and late (ts < W_prev, counted) records
        const bool good = have & ok, late = r.ts + 1u < wm32, kept = good & !late;
        n_bad += (have & !ok) ? 1u : 0u;
        n_late += (good & late) ? 1u : 0u;
        ts_min = sel(kept, min(ts_min, r.ts), ts_min);
        ts_max1 = sel(kept, max(ts_max1, r.ts + 1u), ts_max1);
        surv = kCM2 ? (kept & (r.event == 1u)) : kept;          // WHERE (eventType == 1)
      }
      const uint32_t p = pane30(r.ts, a.pane_m, a.pane_sh);    // floor(ts / S)
      if (kCM2) {
        // warp-ballot stream compaction into the warp's survivor ring
        const uint32_t bal = __ballot_sync(0xffffffffu, surv);
        if (surv) {
          const uint32_t pos = (sv_h + sv_n + __popc(bal & ((1u << lane) - 1u))) & (kSurvCap - 1);
          sv_e[warp][pos] = make_uint4(r.jw0 | ((r.jw2 << 4) & 0xF0F0u), r.jw1, r.cw0, r.cw1);
          sv_p[warp][pos] = p;
        }
        sv_n += __popc(bal);
        if (sv_n >= 32) {
          drain(32);
          sv_n -= 32;
        }
      } else {
        // CM1: reduce per (pane, category) inside the warp
        bool pend = surv;
        const uint32_t s_all = __ballot_sync(0xffffffffu, surv);
        if (s_all) {
          const uint32_t p0 = __shfl_sync(0xffffffffu, p, __ffs(s_all) - 1);
          if (__all_sync(0xffffffffu, !surv || p == p0)) {
            // the usual round: every record in one pane — per category c <= the largest
            // present, one REDUX sum and one ballot count; lane c then adds category c's
            const uint32_t cmax = __reduce_max_sync(0xffffffffu, surv ? r.cat : 0u);
            uint32_t my_s = 0, my_n = 0;
            for (uint32_t c = 0; c <= cmax; c++) {
              const bool me = surv && r.cat == c;
              const uint32_t sc = __reduce_add_sync(0xffffffffu, me ? r.cpu_m : 0u);   // < 32 * 1e7
              const uint32_t nc = __popc(__ballot_sync(0xffffffffu, me));
              my_s = sel((uint32_t)lane == c, sc, my_s);
              my_n = sel((uint32_t)lane == c, nc, my_n);
            }
            if (my_n) {
              if (p0 != c_pane) { c_pane = p0; local_slot(slot_tag, q, p0, c_slot, c_gslot); }
              if (c_gslot == kFail32) n_ovf += my_n;
              else if (c_slot < 2) {
                w_sum[warp][c_slot][lane] += my_s;
                w_cnt[warp][c_slot][lane] += my_n;
              } else {
                const size_t gi = (size_t)c_gslot * q.K + lane;
                atomicAdd(&q.acc_sum[gi], (unsigned long long)my_s);
                atomicAdd(&q.acc_cnt[gi], (unsigned long long)my_n);
              }
            }
            pend = false;
            __syncwarp();   // order lane c's accumulator update before any later leader's
          }
        }
        uint32_t left = __ballot_sync(0xffffffffu, pend);
        while (left) {
          const int leader = __ffs(left) - 1;
          const uint32_t lp = __shfl_sync(0xffffffffu, p, leader);
          const uint32_t lc = __shfl_sync(0xffffffffu, r.cat, leader);
          const bool me = pend && p == lp && r.cat == lc;
          const uint32_t mm = __ballot_sync(0xffffffffu, me);
          const uint32_t sm = __reduce_add_sync(0xffffffffu, me ? r.cpu_m : 0u);   // < 32 * 1e7
          if (lane == leader) {
            if (lp != c_pane) { c_pane = lp; local_slot(slot_tag, q, lp, c_slot, c_gslot); }
            if (c_gslot == kFail32) n_ovf += __popc(mm);
            else if (c_slot < 2) {
              w_sum[warp][c_slot][lc] += sm;
              w_cnt[warp][c_slot][lc] += __popc(mm);
            } else {
              const size_t gi = (size_t)c_gslot * q.K + lc;
              atomicAdd(&q.acc_sum[gi], (unsigned long long)sm);
              atomicAdd(&q.acc_cnt[gi], (unsigned long long)__popc(mm));
            }
          }
          if (me) pend = false;
          left &= ~mm;
          __syncwarp();   // order the leader's smem accumulator update before the next leader's
        }
      }
      if (!__any_sync(0xffffffffu, more)) break;   // warp-local rounds
      // next record of a generic lane: at byte 0 (lane 0), then after each '\n' of the chunk;
      // it ends at the next '\n' of the chunk, else at the first one past the chunk
      have = false;
      if (more) {
        if (pend0) {
          pend0 = false;
          sb = 0u;
          have = pay != 0u;
        } else {
          uint32_t bn;
          if (pop_lowest(n0, n1, n2, n3, bn)) {
            sb = cb + bn + 1u;
            have = sb < pay;
          }
        }
        const uint32_t nn = first_bit128(n0, n1, n2, n3, cb);
        e = sel(nn != 0xFFFFu, nn, e_after);
        more = pend0 || (n0 | n1 | n2 | n3) != 0u;
      }
    }
    __syncwarp();      // stage s and the masks consumed by every lane
    fresh = !geo_cont(geo);
    if (!fresh && lane < 8) {                   // halo masks = the next tile's window bits [0, 256)
      sts32(nl_s + 4 * lane, lds32(nl_s + 4 * (kChunks * 4 + lane)));
      sts32(cm_s + 4 * lane, lds32(cm_s + 4 * (kChunks * 4 + lane)));
    }
    // lanes 24..31 write mask words 128..135 in the next tile's pass 1 (each lane leaves the
    // barrier wait on its own): the halo reads above must be done first
    __syncwarp();
    if (it + kCmStages < ntiles) {
      const uint32_t g2 = cm_issue(iss, st_s, full_s + 8u * s, lane);
      iss.next(a.segs);
      geo0 = s ? geo0 : g2;
      geo1 = s ? g2 : geo1;
    }
  }

  if (kCM2) {
    if (sv_n) drain(sv_n);
  } else {
    __syncthreads();
    if (tid < 20) {
      const int sl = tid / 10, c = tid % 10;
      const unsigned long long tg = slot_tag[sl];
      if (tg != kEmpty64 && (uint32_t)(tg >> 32) != kFail32) {
        unsigned long long sv = 0, cv = 0;
        for (int w = 0; w < kWarps; w++) { sv += w_sum[w][sl][c]; cv += w_cnt[w][sl][c]; }
        if (cv) {
          const size_t gi = (size_t)(tg >> 32) * q.K + c;
          atomicAdd(&q.acc_sum[gi], sv);
          atomicAdd(&q.acc_cnt[gi], cv);
        }
      }
    }
  }
  flush_counters(CtaCounters{n_rec, n_bad, n_late, n_ovf, ts_min, ts_max1}, q.state, &nlm[0][0]);
}

}  // namespace

// Load every kernel of this file now (CUDA 12 loads kernels lazily, at first launch, and a
// lazy load waits for the device: a first launch behind a running spin-wait kernel of another
// handle — the multi-GPU device barriers on a shared GPU — would wait for that spin to time
// out).  Called once per process from lms_query_create.
void preload_cm_kernels() {
  cudaFuncAttributes fa;
  cudaFuncGetAttributes(&fa, k_cm_agg<kCM2S>);
  cudaFuncGetAttributes(&fa, k_cm_agg<kCM1S>);
}

int cm_agg_ctas(const QueryDev& q) {
  static int nsm = -1;
  if (nsm < 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  }
  (void)q;
  return nsm * kCtasPerSm;
}

// cudaFuncSetAttribute once per (kernel, device, size): it is not a per-launch call (and the
// driver may serialise it against running work, which the multi-GPU device-side barriers of
// other handles on the same device must never wait behind).
static cudaError_t set_smem_once(const void* fn, int bytes) {
  static std::mutex mu;
  static const void* done_fn[16];
  static int done_dev[16], done_bytes[16], n_done = 0;
  std::lock_guard<std::mutex> lock(mu);
  int dev = 0;
  cudaGetDevice(&dev);
  for (int i = 0; i < n_done; i++)
    if (done_fn[i] == fn && done_dev[i] == dev && done_bytes[i] >= bytes) return cudaSuccess;
  const cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess && n_done < 16) { done_fn[n_done] = fn; done_dev[n_done] = dev; done_bytes[n_done] = bytes; n_done++; }
  return e;
}

cudaError_t launch_cm_agg(const QueryDev& q, const SegTable& segs, cudaStream_t st) {
  CmArgs a;
  a.q = q;
  a.segs = segs;
  a.total_tiles = segs.tile_prefix[segs.n];
  a.k7f = 0x7F7F7F7Fu;
  a.k256 = 256u;
  a.k512 = 512u;
  pane30_magic(q.S, a.pane_m, a.pane_sh);
  if (a.total_tiles == 0) return cudaSuccess;
  const size_t smem = (size_t)kWarps * kCmStages * kCmStage + kSmemPad;
  const int grid = (int)q.n_agg_ctas;
  cudaError_t e;
  if (q.kind == kCM2S) {
    e = set_smem_once((const void*)k_cm_agg<kCM2S>, (int)smem);
    if (e != cudaSuccess) return e;
    k_cm_agg<kCM2S><<<grid, kCmThreads, smem, st>>>(a);
  } else {
    e = set_smem_once((const void*)k_cm_agg<kCM1S>, (int)smem);
    if (e != cudaSuccess) return e;
    k_cm_agg<kCM1S><<<grid, kCmThreads, smem, st>>>(a);
  }
  return cudaGetLastError();
}

}  // namespace lms
