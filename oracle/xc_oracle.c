/*
 * xc_oracle.c — CPU ORACLE of the XC expert-blob codec (include/spmoe.h,
 * "XC", format SXC5).  TEST INFRASTRUCTURE ONLY: tests/ compare the sm_100a
 * encoder's blob byte for byte against oracle_xc_encode and the decoder's
 * output against the original bits; the product path never links this file.
 *
 * What it restates: the format is this build's (the reference moves raw
 * expert bytes, IoChannel.transfer prefetch.py:45-74), so there is no
 * reference golden vector; parity is pinned by the format's own invariant
 * decode(encode(x)) == x (checked here on CPU too) and by GPU == CPU blob
 * bytes.  Straight-line scalar code in value order:
 *   base   the lowest b <= 240 whose exponent window [b, b+14] holds the
 *          most values; exponent e -> symbol e - b inside it, else 15
 *          (escape, the exponent goes to the block's exception list);
 *   code   symbol histogram -> two-queue Huffman lengths (ties: leaves
 *          before internal nodes, lower ids first) -> lengths capped at
 *          SPMOE_XC_LMAX with the Kraft excess repaid by lengthening the
 *          longest sub-LMAX code (rarest, then highest id) -> canonical
 *          codes in (length, symbol) order, written bit-reversed (LSB
 *          first);
 *   block  4096 values: sign|mantissa bytes; 32 lane substreams of the
 *          codes of values 128 l .. 128 l + 127, bit-contiguous with the
 *          block's run padded to a word (bit mode), or each padded to a
 *          word when the lanes' bit lengths spread over more than 255
 *          (word mode); exception records (index << 8 | exponent) in value
 *          order;
 *   layout header at 0, streams from 512 on 256-byte boundaries in the
 *          order lut (multi-symbol, u32), sm, ex (+ 8 slack bytes), bofs,
 *          lanes, xofs, xrec per segment.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "../include/spmoe.h"

#define LMAX SPMOE_XC_LMAX
#define LANES SPMOE_XC_LANES
#define NSYM SPMOE_XC_NSYM
#define ESC (NSYM - 1)
#define PER_LANE (SPMOE_XC_BLOCK / LANES)

static uint64_t a256(uint64_t x) { return (x + 255) & ~(uint64_t)255; }

/* The segment's base exponent from its exponent histogram. */
uint32_t oracle_xc_base(const uint64_t hist[256]) {
  uint32_t best = 0;
  uint64_t best_mass = 0;
  for (uint32_t b = 0; b + ESC <= 255 && b <= 240; ++b) {
    uint64_t m = 0;
    for (uint32_t e = b; e < b + ESC; ++e) m += hist[e];
    if (m > best_mass) {
      best_mass = m;
      best = b;
    }
  }
  return best;
}

static int sym_of(int e, uint32_t base) { return (e >= (int)base && e < (int)base + ESC) ? e - (int)base : ESC; }

void oracle_xc_code_lengths(const uint64_t cnt[NSYM], uint8_t len[NSYM]) {
  memset(len, 0, NSYM);
  int sym[NSYM], n = 0;
  for (int s = 0; s < NSYM; ++s)
    if (cnt[s]) sym[n++] = s;
  if (n == 0) return;
  if (n == 1) {
    len[sym[0]] = 1;
    return;
  }
  /* leaves sorted by (count asc, id asc): insertion sort, stable */
  for (int i = 1; i < n; ++i) {
    int x = sym[i], j = i - 1;
    while (j >= 0 && cnt[sym[j]] > cnt[x]) {
      sym[j + 1] = sym[j];
      --j;
    }
    sym[j + 1] = x;
  }
  uint64_t w[2 * NSYM];
  int parent[2 * NSYM], depth[2 * NSYM];
  for (int i = 0; i < n; ++i) w[i] = cnt[sym[i]];
  int li = 0, ii = n, next = n;
  for (int k = 0; k < n - 1; ++k) {
    int pick[2];
    for (int t = 0; t < 2; ++t) {
      if (li < n && (ii == next || w[li] <= w[ii])) pick[t] = li++;
      else pick[t] = ii++;
    }
    w[next] = w[pick[0]] + w[pick[1]];
    parent[pick[0]] = parent[pick[1]] = next;
    ++next;
  }
  const int root = 2 * n - 2;
  depth[root] = 0;
  for (int v = root - 1; v >= 0; --v) depth[v] = depth[parent[v]] + 1;
  int maxlen = 0;
  for (int i = 0; i < n; ++i) {
    len[sym[i]] = (uint8_t)depth[i];
    if (depth[i] > maxlen) maxlen = depth[i];
  }
  if (maxlen <= LMAX) return;
  int64_t kraft = 0;
  for (int s = 0; s < NSYM; ++s) {
    if (!len[s]) continue;
    if (len[s] > LMAX) len[s] = LMAX;
    kraft += (int64_t)1 << (LMAX - len[s]);
  }
  while (kraft > ((int64_t)1 << LMAX)) {
    int best = -1;
    for (int s = 0; s < NSYM; ++s) {
      if (!len[s] || len[s] >= LMAX) continue;
      if (best < 0 || len[s] > len[best] ||
          (len[s] == len[best] && (cnt[s] < cnt[best] || (cnt[s] == cnt[best] && s > best))))
        best = s;
    }
    kraft -= (int64_t)1 << (LMAX - len[best] - 1);
    len[best]++;
  }
}

/* canonical codes, bit-reversed for LSB-first packing */
static void rev_codes(const uint8_t len[NSYM], uint16_t rev[NSYM]) {
  memset(rev, 0, sizeof(uint16_t) * NSYM);
  uint32_t code = 0;
  int prev = 0;
  for (int L = 1; L <= LMAX; ++L)
    for (int s = 0; s < NSYM; ++s) {
      if (len[s] != L) continue;
      if (prev) code <<= (L - prev);
      prev = L;
      uint32_t r = 0;
      for (int b = 0; b < L; ++b) r |= ((code >> b) & 1u) << (L - 1 - b);
      rev[s] = (uint16_t)r;
      ++code;
    }
}

/* single-symbol table: entry q (12 peeked bits) = symbol | length << 8 */
void oracle_xc_lut(const uint8_t len[NSYM], uint16_t lut[1 << LMAX]) {
  uint16_t rev[NSYM];
  rev_codes(len, rev);
  memset(lut, 0, sizeof(uint16_t) << LMAX);
  for (int s = 0; s < NSYM; ++s) {
    const int L = len[s];
    if (!L) continue;
    for (uint32_t q = 0; q < (1u << (LMAX - L)); ++q) lut[rev[s] | (q << L)] = (uint16_t)(s | (L << 8));
  }
}

/* Multi-symbol table from the single-symbol one (restates lut2_of in
 * paper_2510_10302_b200/csrc/spmoe_codec.cu): entry q = up to five whole
 * codes that fit in the 12 peeked bits.  An unused pattern of an
 * incomplete code (length 0) still advances by one bit. */
void oracle_xc_lut2(const uint16_t lut[1 << LMAX], uint32_t lut2[1 << LMAX]) {
  for (uint32_t q = 0; q < (1u << LMAX); ++q) {
    const uint32_t e0 = lut[q];
    uint32_t tot = e0 >> 8, cnt = 1, syms = e0 & 0xfu;
    if (tot == 0) tot = 1;
    while (cnt < 5) {
      const uint32_t e = lut[q >> tot], l = e >> 8;
      if (!l || tot + l > LMAX) break;
      syms |= (e & 0xfu) << (4 * cnt);
      ++cnt;
      tot += l;
    }
    lut2[q] = syms | ((4 * cnt) << 20) | (tot << 25);
  }
}

/* Code bits of each lane of block b. */
static void block_lane_bits(const uint16_t* s, int64_t b, const spmoe_xc_segment* g, uint32_t lb[LANES]) {
  for (int l = 0; l < LANES; ++l) {
    uint32_t bits = 0;
    for (int j = 0; j < PER_LANE; ++j) bits += g->len[sym_of((s[b * SPMOE_XC_BLOCK + l * PER_LANE + j] >> 7) & 0xff, g->base)];
    lb[l] = bits;
  }
}

/* Word mode when the lane lengths spread over more than 255 bits. */
static int block_word_mode(const uint32_t lb[LANES]) {
  uint32_t lo = lb[0], hi = lb[0];
  for (int l = 1; l < LANES; ++l) {
    if (lb[l] < lo) lo = lb[l];
    if (lb[l] > hi) hi = lb[l];
  }
  return hi - lo > 255;
}

static uint32_t block_words(const uint32_t lb[LANES]) {
  uint32_t w = 0, bits = 0;
  for (int l = 0; l < LANES; ++l) {
    w += (lb[l] + 31) / 32;
    bits += lb[l];
  }
  return block_word_mode(lb) ? w : (bits + 31) / 32;
}

/* Encode nseg segments (back to back in src).  Returns the blob size; the
 * blob is written only if out != NULL and cap >= size.  0 on invalid
 * segment sizes. */
uint64_t oracle_xc_encode(const uint16_t* src, int nseg, const int64_t* seg_n, uint8_t* out, uint64_t cap,
                          spmoe_xc_header* hdr_out) {
  if (nseg < 1 || nseg > SPMOE_XC_MAX_SEG) return 0;
  for (int i = 0; i < nseg; ++i)
    if (seg_n[i] <= 0 || seg_n[i] % SPMOE_XC_BLOCK) return 0;
  spmoe_xc_header hdr;
  memset(&hdr, 0, sizeof(hdr));
  hdr.magic = SPMOE_XC_MAGIC;
  hdr.nseg = (uint32_t)nseg;
  uint16_t revs[SPMOE_XC_MAX_SEG][NSYM];
  /* pass 1: base, codes, sizes, layout */
  const uint16_t* s = src;
  uint64_t pos = a256(sizeof(spmoe_xc_header)), raw = 0;
  for (int i = 0; i < nseg; ++i) {
    spmoe_xc_segment* g = &hdr.seg[i];
    const int64_t n = seg_n[i], nb = n / SPMOE_XC_BLOCK;
    uint64_t hist[256], cnt[NSYM];
    memset(hist, 0, sizeof(hist));
    memset(cnt, 0, sizeof(cnt));
    for (int64_t k = 0; k < n; ++k) hist[(s[k] >> 7) & 0xff]++;
    g->base = oracle_xc_base(hist);
    for (int e = 0; e < 256; ++e) cnt[sym_of(e, g->base)] += hist[e];
    oracle_xc_code_lengths(cnt, g->len);
    rev_codes(g->len, revs[i]);
    g->n = (uint64_t)n;
    g->n_exc = (uint32_t)cnt[ESC];
    uint64_t words = 0;
    for (int64_t b = 0; b < nb; ++b) {
      uint32_t lb[LANES];
      block_lane_bits(s, b, g, lb);
      words += block_words(lb);
    }
    g->ex_words = (uint32_t)words;
    g->off_lut = pos; pos = a256(pos + (4u << LMAX));
    g->off_sm = pos; pos = a256(pos + (uint64_t)n);
    g->off_ex = pos; pos = a256(pos + words * 4 + 8);
    g->off_bofs = pos; pos = a256(pos + (uint64_t)(nb + 1) * 4);
    g->off_lanes = pos; pos = a256(pos + (uint64_t)nb * LANES);
    g->off_lbase = pos; pos = a256(pos + (uint64_t)nb * 2);
    g->off_xofs = pos; pos = a256(pos + (uint64_t)(nb + 1) * 4);
    g->off_xrec = pos; pos = a256(pos + (uint64_t)g->n_exc * 4);
    raw += 2 * (uint64_t)n;
    s += n;
  }
  hdr.blob_bytes = pos;
  hdr.raw_bytes = raw;
  if (hdr_out) *hdr_out = hdr;
  if (!out || cap < pos) return pos;
  /* pass 2: streams */
  memset(out, 0, pos);
  memcpy(out, &hdr, sizeof(hdr));
  s = src;
  for (int i = 0; i < nseg; ++i) {
    const spmoe_xc_segment* g = &hdr.seg[i];
    const int64_t n = (int64_t)g->n, nb = n / SPMOE_XC_BLOCK;
    uint16_t lut1[1 << LMAX];
    oracle_xc_lut(g->len, lut1);
    oracle_xc_lut2(lut1, (uint32_t*)(out + g->off_lut));
    uint8_t* sm = out + g->off_sm;
    uint32_t* ex = (uint32_t*)(out + g->off_ex);
    uint32_t* bofs = (uint32_t*)(out + g->off_bofs);
    uint8_t* lanes = out + g->off_lanes;
    uint32_t* xofs = (uint32_t*)(out + g->off_xofs);
    uint32_t* xrec = (uint32_t*)(out + g->off_xrec);
    uint16_t* lbase = (uint16_t*)(out + g->off_lbase);
    uint32_t w = 0, x = 0;
    for (int64_t b = 0; b < nb; ++b) {
      bofs[b] = w;
      xofs[b] = x;
      uint32_t lb[LANES];
      block_lane_bits(s, b, g, lb);
      const int wm = block_word_mode(lb);
      uint32_t lo = lb[0];
      for (int l = 1; l < LANES; ++l)
        if (lb[l] < lo) lo = lb[l];
      lbase[b] = (uint16_t)(wm ? 0x8000u : lo);
      uint64_t bitpos = (uint64_t)w * 32; /* the lane's first bit within ex */
      for (int l = 0; l < LANES; ++l) {
        lanes[b * LANES + l] = (uint8_t)(wm ? (lb[l] + 31) / 32 : lb[l] - lo);
        for (int j = 0; j < PER_LANE; ++j) {
          const int64_t k = b * SPMOE_XC_BLOCK + l * PER_LANE + j;
          const uint16_t v = s[k];
          const int e = (v >> 7) & 0xff, y = sym_of(e, g->base);
          sm[k] = (uint8_t)(((v >> 8) & 0x80) | (v & 0x7f));
          if (y == ESC) xrec[x++] = ((uint32_t)(l * PER_LANE + j) << 8) | (uint32_t)e;
          for (int t = 0; t < g->len[y]; ++t, ++bitpos)
            if ((revs[i][y] >> t) & 1u) ex[bitpos >> 5] |= 1u << (bitpos & 31);
        }
        if (wm) bitpos = (bitpos + 31) & ~(uint64_t)31;
      }
      w += block_words(lb);
    }
    bofs[nb] = w;
    xofs[nb] = x;
    s += n;
  }
  return pos;
}

/* Decode a blob into dst (raw_bytes / 2 values).  0 ok, 1 bad blob. */
int oracle_xc_decode(const uint8_t* blob, uint16_t* dst) {
  spmoe_xc_header hdr;
  memcpy(&hdr, blob, sizeof(hdr));
  if (hdr.magic != SPMOE_XC_MAGIC || hdr.nseg < 1 || hdr.nseg > SPMOE_XC_MAX_SEG) return 1;
  uint16_t* d = dst;
  for (uint32_t i = 0; i < hdr.nseg; ++i) {
    const spmoe_xc_segment* g = &hdr.seg[i];
    const int64_t n = (int64_t)g->n, nb = n / SPMOE_XC_BLOCK;
    if (n <= 0 || n % SPMOE_XC_BLOCK || g->base > 240) return 1;
    uint16_t lut[1 << LMAX];  /* the decoder walks the single-symbol table built from len[] */
    oracle_xc_lut(g->len, lut);
    const uint8_t* sm = blob + g->off_sm;
    const uint32_t* ex = (const uint32_t*)(blob + g->off_ex);
    const uint32_t* bofs = (const uint32_t*)(blob + g->off_bofs);
    const uint8_t* lanes = blob + g->off_lanes;
    const uint32_t* xofs = (const uint32_t*)(blob + g->off_xofs);
    const uint32_t* xrec = (const uint32_t*)(blob + g->off_xrec);
    const uint16_t* lbase = (const uint16_t*)(blob + g->off_lbase);
    for (int64_t b = 0; b < nb; ++b) {
      uint32_t x = xofs[b];
      const int wm = lbase[b] >> 15;
      uint64_t bitpos = (uint64_t)bofs[b] * 32;
      for (int l = 0; l < LANES; ++l) {
        const uint32_t lane_bits = wm ? 32u * lanes[b * LANES + l] : (uint32_t)(lbase[b] & 0x7fff) + lanes[b * LANES + l];
        const uint64_t end = bitpos + lane_bits;
        for (int j = 0; j < PER_LANE; ++j) {
          uint32_t peek = 0; /* the next LMAX bits, LSB first */
          for (int t = 0; t < LMAX; ++t) {
            const uint64_t q = bitpos + t;
            if (q < (uint64_t)bofs[b + 1] * 32) peek |= ((ex[q >> 5] >> (q & 31)) & 1u) << t;
          }
          const uint16_t e = lut[peek];
          const int L = e >> 8;
          if (L == 0) return 1;
          bitpos += L;
          const int64_t k = b * SPMOE_XC_BLOCK + l * PER_LANE + j;
          uint32_t expo = g->base + (e & 0xfu);
          if ((e & 0xfu) == ESC) {
            if (x >= xofs[b + 1] || (xrec[x] >> 8) != (uint32_t)(l * PER_LANE + j)) return 1;
            expo = xrec[x++] & 0xffu;
          }
          const uint8_t bb = sm[k];
          d[k] = (uint16_t)(((bb & 0x80) << 8) | (expo << 7) | (bb & 0x7f));
        }
        if (bitpos > end) return 1;
        bitpos = end;
      }
      if ((bitpos + 31) / 32 > bofs[b + 1]) return 1;
      if (x != xofs[b + 1]) return 1;
    }
    d += n;
  }
  return 0;
}
