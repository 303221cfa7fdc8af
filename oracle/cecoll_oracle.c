/*
 * cecoll oracle — TEST INFRASTRUCTURE ONLY (see cecoll_oracle.h).
 *
 * Every function cites the reference file:line it restates. Paths are
 * relative to /root/reference/proj.
 */
#include "cecoll_oracle.h"

#include <pthread.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

ora_program* ora_program_new(void) { return (ora_program*)calloc(1, sizeof(ora_program)); }
void ora_program_free(ora_program* p) { free(p); }

/* compiler.cpp:8-20 */
const char* ora_impl_name(int impl) {
  switch (impl) {
    case ORA_PCPY: return "pcpy";
    case ORA_BCST: return "bcst";
    case ORA_SWAP: return "swap";
    case ORA_B2B: return "b2b";
    case ORA_PRELAUNCH_PCPY: return "prelaunch_pcpy";
    case ORA_PRELAUNCH_BCST: return "prelaunch_bcst";
    case ORA_PRELAUNCH_SWAP: return "prelaunch_swap";
    case ORA_PRELAUNCH_B2B: return "prelaunch_b2b";
  }
  return "?";
}

/* compiler.cpp:22-37 ("baseline" aliases pcpy, line 25) */
int ora_parse_impl(const char* name) {
  if (strcmp(name, "baseline") == 0) return ORA_PCPY;
  for (int i = 0; i < 8; ++i)
    if (strcmp(name, ora_impl_name(i)) == 0) return i;
  return -1;
}

static int is_prelaunched(int impl) { return impl >= ORA_PRELAUNCH_PCPY; }
static int base_of(int impl) { return is_prelaunched(impl) ? impl - 4 : impl; }

/* compiler.cpp:70-75 */
int ora_valid_for(int impl, int kind) {
  int base = base_of(impl);
  if (base == ORA_BCST) return kind == ORA_ALLGATHER;
  if (base == ORA_SWAP) return kind == ORA_ALLTOALL;
  return 1;
}

/* Builder (compiler.cpp:93-113): queues opened per GPU in ascending engine
 * order, each sealed with an AtomicSignal on the next signal slot. */
typedef struct {
  ora_program* p;
  int next_engine[ORA_MAX_QUEUES];
  int next_signal;
} builder;

static ora_queue* open_queue(builder* b, int gpu) {
  ora_queue* q = &b->p->queues[b->p->nqueues++];
  memset(q, 0, sizeof(*q));
  q->gpu = gpu;
  q->engine = b->next_engine[gpu]++;
  q->doorbell_count = 1;
  return q;
}

static void seal_queue(builder* b, ora_queue* q) {
  ora_cmd* c = &q->cmds[q->ncmds++];
  memset(c, 0, sizeof(*c));
  c->kind = ORA_SIGNAL;
  c->signal_target = b->next_signal++;
  c->poll_slot = -1;
}

static ora_cmd* push_cmd(ora_queue* q, int kind) {
  ora_cmd* c = &q->cmds[q->ncmds++];
  memset(c, 0, sizeof(*c));
  c->kind = kind;
  c->signal_target = -1;
  c->poll_slot = -1;
  return c;
}

/* ag_src / out_slot / aa_src (compiler.cpp:115-126) */
static ora_ref ag_src(const ora_program* p, int gpu) {
  ora_ref r = {gpu, ORA_INPUT, 0, p->chunk_size};
  return r;
}
static ora_ref out_slot(const ora_program* p, int gpu, int slot) {
  ora_ref r = {gpu, p->in_place ? ORA_INPUT : ORA_OUTPUT, slot * p->chunk_size, p->chunk_size};
  return r;
}
static ora_ref aa_src(const ora_program* p, int gpu, int chunk) {
  ora_ref r = {gpu, ORA_INPUT, chunk * p->chunk_size, p->chunk_size};
  return r;
}

/* compile_pcpy (compiler.cpp:139-164): per GPU i, lane d=1..n-1 targets
 * j=(i+d)%n with one copy and one signal on its own engine. */
static int compile_pcpy(ora_program* p, int engines) {
  if (p->in_place) return ORA_EINVAL;
  if (engines < p->gpu_count - 1) return ORA_EINVAL;
  builder b;
  memset(&b, 0, sizeof(b));
  b.p = p;
  const int n = p->gpu_count;
  for (int i = 0; i < n; ++i)
    for (int d = 1; d < n; ++d) {
      const int j = (i + d) % n;
      ora_queue* q = open_queue(&b, i);
      ora_cmd* c = push_cmd(q, ORA_COPY);
      c->src = p->kind == ORA_ALLGATHER ? ag_src(p, i) : aa_src(p, i, j);
      c->dst = out_slot(p, j, i);
      c->size = p->chunk_size;
      seal_queue(&b, q);
    }
  return ORA_OK;
}

/* compile_bcst (compiler.cpp:166-205): floor((n-1)/2) broadcasts to peers
 * (i+2k+1)%n, (i+2k+2)%n, plus a copy to (i+n-1)%n when n is even. */
static int compile_bcst(ora_program* p, int engines) {
  if (p->kind == ORA_ALLTOALL) return ORA_EINVAL;
  const int n = p->gpu_count;
  const int broadcasts = (n - 1) / 2;
  const int leftover = (n % 2) == 0;
  if (engines < broadcasts + (leftover ? 1 : 0)) return ORA_EINVAL;
  builder b;
  memset(&b, 0, sizeof(b));
  b.p = p;
  for (int i = 0; i < n; ++i) {
    for (int k = 0; k < broadcasts; ++k) {
      ora_queue* q = open_queue(&b, i);
      ora_cmd* c = push_cmd(q, ORA_BROADCAST);
      c->src = ag_src(p, i);
      c->dst = out_slot(p, (i + 2 * k + 1) % n, i);
      c->dst2 = out_slot(p, (i + 2 * k + 2) % n, i);
      c->size = p->chunk_size;
      seal_queue(&b, q);
    }
    if (leftover) {
      ora_queue* q = open_queue(&b, i);
      ora_cmd* c = push_cmd(q, ORA_COPY);
      c->src = ag_src(p, i);
      c->dst = out_slot(p, (i + n - 1) % n, i);
      c->size = p->chunk_size;
      seal_queue(&b, q);
    }
  }
  return ORA_OK;
}

/* compile_swap (compiler.cpp:207-239): in-place; pair (i<j) owned by i when
 * j-i <= n/2 else by j; owners issue their swaps in ascending peer order of
 * the pair enumeration (i ascending, then j ascending). */
static int compile_swap(ora_program* p, int engines) {
  p->in_place = 1;
  if (p->kind != ORA_ALLTOALL) return ORA_EINVAL;
  const int n = p->gpu_count;
  if (engines < (n - 1 + 1) / 2) return ORA_EINVAL;
  builder b;
  memset(&b, 0, sizeof(b));
  b.p = p;
  for (int g = 0; g < n; ++g)
    for (int i = 0; i < n; ++i)
      for (int j = i + 1; j < n; ++j) {
        const int owner = (j - i) <= n / 2 ? i : j;
        if (owner != g) continue;
        const int peer = owner == i ? j : i;
        ora_queue* q = open_queue(&b, g);
        ora_cmd* c = push_cmd(q, ORA_SWAPCMD);
        c->src = aa_src(p, g, peer);
        c->peer = aa_src(p, peer, g);
        c->size = p->chunk_size;
        seal_queue(&b, q);
      }
  return ORA_OK;
}

/* compile_b2b (compiler.cpp:241-265): one queue per GPU, n-1 copies in the
 * pcpy rotation, one trailing signal. */
static int compile_b2b(ora_program* p) {
  if (p->in_place) return ORA_EINVAL;
  builder b;
  memset(&b, 0, sizeof(b));
  b.p = p;
  const int n = p->gpu_count;
  for (int i = 0; i < n; ++i) {
    ora_queue* q = open_queue(&b, i);
    for (int d = 1; d < n; ++d) {
      const int j = (i + d) % n;
      ora_cmd* c = push_cmd(q, ORA_COPY);
      c->src = p->kind == ORA_ALLGATHER ? ag_src(p, i) : aa_src(p, i, j);
      c->dst = out_slot(p, j, i);
      c->size = p->chunk_size;
    }
    seal_queue(&b, q);
  }
  return ORA_OK;
}

/* apply_prelaunch (compiler.cpp:267-285): a Poll on slot 100000+k
 * (expected 1) is prepended to every nonempty queue. */
static void apply_prelaunch(ora_program* p) {
  int slot = 100000;
  for (int qi = 0; qi < p->nqueues; ++qi) {
    ora_queue* q = &p->queues[qi];
    if (q->ncmds == 0) continue;
    memmove(&q->cmds[1], &q->cmds[0], sizeof(ora_cmd) * (size_t)q->ncmds);
    memset(&q->cmds[0], 0, sizeof(ora_cmd));
    q->cmds[0].kind = ORA_POLL;
    q->cmds[0].poll_slot = slot++;
    q->cmds[0].signal_target = -1;
    q->cmds[0].expected_value = 1;
    q->ncmds++;
  }
  p->prelaunched = 1;
}

/* compile (compiler.cpp:287-303) + validate_spec (program.cpp:31-38). */
int ora_compile(int impl, int kind, int64_t chunk_size, int n, int engines, ora_program* p) {
  memset(p, 0, offsetof(ora_program, queues));
  if (impl < 0 || impl > 7 || (kind != ORA_ALLGATHER && kind != ORA_ALLTOALL)) return ORA_EINVAL;
  if (!ora_valid_for(impl, kind)) return ORA_EINVAL;
  if (chunk_size <= 0 || n < 2) return ORA_EINVAL;
  if (n > 32 || (int64_t)n * (n - 1) > ORA_MAX_QUEUES) return ORA_EINVAL; /* oracle capacity */
  p->kind = kind;
  p->chunk_size = chunk_size;
  p->gpu_count = n;
  p->impl = impl;
  p->in_place = base_of(impl) == ORA_SWAP;
  int rc;
  switch (base_of(impl)) {
    case ORA_PCPY: rc = compile_pcpy(p, engines); break;
    case ORA_BCST: rc = compile_bcst(p, engines); break;
    case ORA_SWAP: rc = compile_swap(p, engines); break;
    default: rc = compile_b2b(p); break;
  }
  if (rc != ORA_OK) return rc;
  if (is_prelaunched(impl)) apply_prelaunch(p);
  return ORA_OK;
}

/* dump_program (program.cpp:205-254) */
static int ref_str(char* out, size_t cap, const ora_ref* r) {
  return snprintf(out, cap, "g%d%s%lld+%lld]", r->gpu, r->buffer == ORA_INPUT ? ".in[" : ".out[",
                  (long long)r->offset, (long long)r->length);
}

int64_t ora_dump(const ora_program* p, char* buf, size_t cap) {
  static const char* names[] = {"copy", "broadcast", "swap", "signal", "poll", "timestamp"};
  size_t pos = 0;
  char a[96], b[96], c[96];
#define EMIT(...)                                                  \
  do {                                                             \
    int k_ = snprintf(buf + pos, pos < cap ? cap - pos : 0, __VA_ARGS__); \
    pos += (size_t)k_;                                             \
  } while (0)
  for (int qi = 0; qi < p->nqueues; ++qi) {
    const ora_queue* q = &p->queues[qi];
    for (int ci = 0; ci < q->ncmds; ++ci) {
      const ora_cmd* cmd = &q->cmds[ci];
      EMIT("q%d(g%de%d)\t%d\t%s\t", qi, q->gpu, q->engine, ci, names[cmd->kind]);
      switch (cmd->kind) {
        case ORA_COPY:
          ref_str(a, sizeof a, &cmd->src);
          ref_str(b, sizeof b, &cmd->dst);
          EMIT("%s\t%s\t%lld\t-", a, b, (long long)cmd->size);
          break;
        case ORA_BROADCAST:
          ref_str(a, sizeof a, &cmd->src);
          ref_str(b, sizeof b, &cmd->dst);
          ref_str(c, sizeof c, &cmd->dst2);
          EMIT("%s\t%s,%s\t%lld\t-", a, b, c, (long long)cmd->size);
          break;
        case ORA_SWAPCMD:
          ref_str(a, sizeof a, &cmd->src);
          ref_str(b, sizeof b, &cmd->peer);
          EMIT("%s\t%s\t%lld\t-", a, b, (long long)cmd->size);
          break;
        case ORA_SIGNAL: EMIT("-\t-\t0\t%d", cmd->signal_target); break;
        case ORA_POLL: EMIT("-\t-\t0\t%d", cmd->poll_slot); break;
        default: EMIT("-\t-\t0\t-"); break;
      }
      EMIT("\n");
    }
  }
#undef EMIT
  if (pos >= cap) return ORA_ENOSPC;
  return (int64_t)pos;
}

static int is_data(int kind) { return kind == ORA_COPY || kind == ORA_BROADCAST || kind == ORA_SWAPCMD; }

/* static_metrics (program.cpp:40-65) */
void ora_static_metrics(const ora_program* p, ora_metrics* m) {
  memset(m, 0, sizeof(*m));
  for (int qi = 0; qi < p->nqueues; ++qi) {
    const ora_queue* q = &p->queues[qi];
    if (q->ncmds == 0) continue;
    m->engines_used += 1;
    m->doorbells += q->doorbell_count;
    for (int ci = 0; ci < q->ncmds; ++ci) {
      int k = q->cmds[ci].kind;
      if (is_data(k)) m->data_commands++;
      else if (k == ORA_SIGNAL) m->sync_commands++;
      else if (k == ORA_POLL) m->poll_commands++;
    }
  }
}

/* account_traffic (verifier.cpp:281-327) */
void ora_traffic(const ora_program* p, int64_t* tr, int64_t* tw, int64_t* tl, int64_t* gr, int64_t* gw) {
  *tr = *tw = *tl = 0;
  if (gr) memset(gr, 0, sizeof(int64_t) * (size_t)p->gpu_count);
  if (gw) memset(gw, 0, sizeof(int64_t) * (size_t)p->gpu_count);
#define RD(g, v) do { *tr += (v); if (gr) gr[g] += (v); } while (0)
#define WR(g, v) do { *tw += (v); if (gw) gw[g] += (v); } while (0)
  for (int qi = 0; qi < p->nqueues; ++qi) {
    const ora_queue* q = &p->queues[qi];
    for (int ci = 0; ci < q->ncmds; ++ci) {
      const ora_cmd* c = &q->cmds[ci];
      switch (c->kind) {
        case ORA_COPY:
          RD(c->src.gpu, c->size);
          WR(c->dst.gpu, c->size);
          if (c->src.gpu != c->dst.gpu) *tl += c->size;
          break;
        case ORA_BROADCAST:
          RD(c->src.gpu, c->size);
          WR(c->dst.gpu, c->size);
          WR(c->dst2.gpu, c->size);
          if (c->src.gpu != c->dst.gpu) *tl += c->size;
          if (c->src.gpu != c->dst2.gpu) *tl += c->size;
          break;
        case ORA_SWAPCMD:
          RD(c->src.gpu, c->size);
          RD(c->peer.gpu, c->size);
          WR(c->src.gpu, c->size);
          WR(c->peer.gpu, c->size);
          *tl += 2 * c->size;
          break;
        default: break;
      }
    }
  }
#undef RD
#undef WR
}

/* ---- symbolic verifier (verifier.cpp:11-279) ---- */

typedef struct { int origin, chunk; } label;
typedef struct { label cur, init; int written; } slot;

typedef struct {
  const ora_program* p;
  int n, in_chunks;
  slot* input;  /* [gpu][in_chunks]; in-place: [gpu][n] */
  slot* output; /* [gpu][n]; NULL when in_place */
} symstate;

/* SymbolicState ctor (verifier.cpp:31-47): local chunk pre-placed in slot g. */
static void sym_init(symstate* s, const ora_program* p) {
  s->p = p;
  s->n = p->gpu_count;
  s->in_chunks = p->kind == ORA_ALLGATHER ? 1 : s->n;
  for (int g = 0; g < s->n; ++g) {
    for (int c = 0; c < s->in_chunks; ++c) {
      slot* sl = &s->input[g * s->n + c];
      sl->cur.origin = g; sl->cur.chunk = c;
      sl->init = sl->cur;
      sl->written = 0;
    }
    if (!p->in_place) {
      for (int k = 0; k < s->n; ++k) {
        slot* sl = &s->output[g * s->n + k];
        sl->cur.origin = -1; sl->cur.chunk = -1;
        sl->init = sl->cur;
        sl->written = 0;
      }
      slot* loc = &s->output[g * s->n + g];
      loc->cur.origin = g;
      loc->cur.chunk = p->kind == ORA_ALLGATHER ? 0 : g;
      loc->init = loc->cur;
    }
  }
}

static slot* sym_buf(symstate* s, const ora_ref* r) {
  if (s->p->in_place || r->buffer == ORA_INPUT) return &s->input[r->gpu * s->n];
  return &s->output[r->gpu * s->n];
}

/* Executor::read (verifier.cpp:77-93): reading an overwritten region whose
 * label differs from its initial one is a hazard. */
static int sym_read(symstate* s, const ora_ref* r, label* out, int* cnt) {
  slot* b = sym_buf(s, r);
  int first = (int)(r->offset / s->p->chunk_size), count = (int)(r->length / s->p->chunk_size);
  *cnt = 0;
  for (int c = first; c < first + count; ++c) {
    slot* sl = &b[c];
    if (sl->written && !(sl->cur.origin == sl->init.origin && sl->cur.chunk == sl->init.chunk)) return 0;
    out[(*cnt)++] = sl->cur;
  }
  return 1;
}

static void sym_write(symstate* s, const ora_ref* r, const label* lab, int cnt) {
  slot* b = sym_buf(s, r);
  int first = (int)(r->offset / s->p->chunk_size);
  for (int c = 0; c < cnt; ++c) {
    b[first + c].cur = lab[c];
    b[first + c].written = 1;
  }
}

/* Executor::execute (verifier.cpp:104-141) */
static int sym_exec(symstate* s, const ora_cmd* c) {
  label a[64], b2[64];
  int na, nb;
  switch (c->kind) {
    case ORA_COPY:
      if (!sym_read(s, &c->src, a, &na)) return 0;
      sym_write(s, &c->dst, a, na);
      return 1;
    case ORA_BROADCAST:
      if (!sym_read(s, &c->src, a, &na)) return 0;
      sym_write(s, &c->dst, a, na);
      sym_write(s, &c->dst2, a, na);
      return 1;
    case ORA_SWAPCMD:
      if (!sym_read(s, &c->src, a, &na)) return 0;
      if (!sym_read(s, &c->peer, b2, &nb)) return 0;
      sym_write(s, &c->src, b2, nb);
      sym_write(s, &c->peer, a, na);
      return 1;
    default: return 1;
  }
}

/* Executor::check_postcondition (verifier.cpp:143-169) */
static int sym_post(symstate* s) {
  for (int g = 0; g < s->n; ++g) {
    slot* out = s->p->in_place ? &s->input[g * s->n] : &s->output[g * s->n];
    for (int k = 0; k < s->n; ++k) {
      label l = out[k].cur;
      int good = l.origin >= 0 && l.origin == k;
      if (s->p->kind == ORA_ALLTOALL) good = good && l.chunk == g;
      if (!good) return 0;
    }
  }
  return 1;
}

static uint64_t mt_next(uint64_t* st) { /* xorshift64*: seeded shuffle source */
  uint64_t x = *st;
  x ^= x >> 12; x ^= x << 25; x ^= x >> 27;
  *st = x;
  return x * 0x2545F4914F6CDD1DULL;
}

/* verify_collective (verifier.cpp:239-279), random-interleaving branch. */
int ora_verify(const ora_program* p, int trials, uint64_t seed) {
  const int n = p->gpu_count;
  int total = 0;
  for (int qi = 0; qi < p->nqueues; ++qi)
    for (int ci = 0; ci < p->queues[qi].ncmds; ++ci) total += is_data(p->queues[qi].cmds[ci].kind);
  if (total == 0) return ORA_VERDICT_MISMATCH;
  symstate s;
  s.input = (slot*)calloc((size_t)n * n, sizeof(slot));
  s.output = (slot*)calloc((size_t)n * n, sizeof(slot));
  int* cursor = (int*)calloc((size_t)p->nqueues, sizeof(int));
  int* pending = (int*)calloc((size_t)p->nqueues, sizeof(int));
  uint64_t st = seed * 0x9E3779B97F4A7C15ULL + 1;
  int verdict = ORA_VERDICT_OK;
  for (int t = 0; t <= trials && verdict == ORA_VERDICT_OK; ++t) {
    sym_init(&s, p);
    int np = 0;
    for (int qi = 0; qi < p->nqueues; ++qi) {
      cursor[qi] = 0;
      if (p->queues[qi].ncmds) pending[np++] = qi;
    }
    while (np > 0) {
      /* trial 0 runs the program order; later trials pick a random queue */
      int k = t == 0 ? 0 : (int)(mt_next(&st) % (uint64_t)np);
      int qi = pending[k];
      const ora_queue* q = &p->queues[qi];
      const ora_cmd* c = &q->cmds[cursor[qi]++];
      if (!sym_exec(&s, c)) { verdict = ORA_VERDICT_HAZARD; break; }
      if (cursor[qi] == q->ncmds) {
        if (t == 0) { memmove(&pending[0], &pending[1], sizeof(int) * (size_t)(np - 1)); np--; }
        else pending[k] = pending[--np];
      }
    }
    if (verdict == ORA_VERDICT_OK && !sym_post(&s)) verdict = ORA_VERDICT_MISMATCH;
  }
  free(s.input); free(s.output); free(cursor); free(pending);
  return verdict;
}

/* select_implementation (compiler.cpp:305-318) */
int ora_select(int kind, int64_t size) {
  if (size < (1LL << 10)) return -1;
  if (kind == ORA_ALLGATHER) {
    if (size < (256LL << 10)) return ORA_PRELAUNCH_B2B;
    if (size < (1LL << 20)) return ORA_PRELAUNCH_BCST;
    if (size < (512LL << 20)) return ORA_PRELAUNCH_PCPY;
    return ORA_PCPY;
  }
  if (size < (64LL << 10)) return ORA_PRELAUNCH_B2B;
  if (size < (4LL << 20)) return ORA_PRELAUNCH_SWAP;
  if (size < (1LL << 30)) return ORA_PRELAUNCH_PCPY;
  return ORA_PCPY;
}

/* ---- byte level ---- */

static uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ULL;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
  return x ^ (x >> 31);
}

void ora_fill_pattern(uint8_t* buf, int64_t bytes, int rank, uint64_t seed) {
  const uint64_t base = seed ^ ((uint64_t)rank << 48);
  int64_t words = bytes / 8;
  for (int64_t w = 0; w < words; ++w) {
    uint64_t v = splitmix64(base ^ (uint64_t)w);
    memcpy(buf + 8 * w, &v, 8);
  }
  if (bytes % 8) {
    uint64_t v = splitmix64(base ^ (uint64_t)words);
    memcpy(buf + 8 * words, &v, (size_t)(bytes % 8));
  }
}

static uint8_t* byte_region(const ora_program* p, uint8_t* const* in, uint8_t* const* out, const ora_ref* r) {
  uint8_t* base = (p->in_place || r->buffer == ORA_INPUT) ? in[r->gpu] : out[r->gpu];
  return base + r->offset;
}

/* Byte execution of the command semantics (verifier.cpp:104-141) after the
 * local placement of verifier.cpp:40-44. Swap exchanges through a bounce
 * buffer so both sides observe the pre-swap contents. */
int ora_execute(const ora_program* p, uint8_t* const* in, uint8_t* const* out) {
  const int n = p->gpu_count;
  const int64_t s = p->chunk_size;
  if (!p->in_place)
    for (int g = 0; g < n; ++g)
      memcpy(out[g] + (int64_t)g * s, in[g] + (p->kind == ORA_ALLGATHER ? 0 : (int64_t)g * s), (size_t)s);
  uint8_t* tmp = NULL;
  for (int qi = 0; qi < p->nqueues; ++qi) {
    const ora_queue* q = &p->queues[qi];
    for (int ci = 0; ci < q->ncmds; ++ci) {
      const ora_cmd* c = &q->cmds[ci];
      switch (c->kind) {
        case ORA_COPY:
          memcpy(byte_region(p, in, out, &c->dst), byte_region(p, in, out, &c->src), (size_t)c->size);
          break;
        case ORA_BROADCAST: {
          const uint8_t* src = byte_region(p, in, out, &c->src);
          memcpy(byte_region(p, in, out, &c->dst), src, (size_t)c->size);
          memcpy(byte_region(p, in, out, &c->dst2), src, (size_t)c->size);
          break;
        }
        case ORA_SWAPCMD: {
          if (!tmp) tmp = (uint8_t*)malloc((size_t)s);
          uint8_t* a = byte_region(p, in, out, &c->src);
          uint8_t* b = byte_region(p, in, out, &c->peer);
          memcpy(tmp, a, (size_t)c->size);
          memcpy(a, b, (size_t)c->size);
          memcpy(b, tmp, (size_t)c->size);
          break;
        }
        default: break;
      }
    }
  }
  free(tmp);
  return ORA_OK;
}

/* Byte postcondition (verifier.cpp:143-169): AG out_g[k] == in_k[0,s);
 * AA out_g[k] == in_k[g*s, (g+1)*s). */
int64_t ora_check(int kind, int64_t s, int n, int in_place, uint8_t* const* orig, uint8_t* const* res) {
  (void)in_place;
  for (int g = 0; g < n; ++g)
    for (int k = 0; k < n; ++k) {
      const uint8_t* want = orig[k] + (kind == ORA_ALLGATHER ? 0 : (int64_t)g * s);
      if (memcmp(res[g] + (int64_t)k * s, want, (size_t)s) != 0) return (int64_t)g * n + k;
    }
  return -1;
}

typedef struct {
  int kind, n, g0, g1;
  int64_t s;
  uint8_t* const* in;
  uint8_t* const* out;
} rr_arg;

static void* rr_worker(void* v) {
  rr_arg* a = (rr_arg*)v;
  for (int g = a->g0; g < a->g1; ++g)
    for (int k = 0; k < a->n; ++k)
      memcpy(a->out[g] + (int64_t)k * a->s, a->in[k] + (a->kind == ORA_ALLGATHER ? 0 : (int64_t)g * a->s),
             (size_t)a->s);
  return NULL;
}

/* The collective's definition, one destination rank per thread. */
void ora_reference_result(int kind, int64_t s, int n, uint8_t* const* in, uint8_t* const* out, int nthreads) {
  if (nthreads < 1) nthreads = 1;
  if (nthreads > n) nthreads = n;
  pthread_t th[64];
  rr_arg args[64];
  for (int t = 0; t < nthreads; ++t) {
    args[t].kind = kind; args[t].n = n; args[t].s = s; args[t].in = in; args[t].out = out;
    args[t].g0 = n * t / nthreads;
    args[t].g1 = n * (t + 1) / nthreads;
    if (nthreads == 1) rr_worker(&args[t]);
    else pthread_create(&th[t], NULL, rr_worker, &args[t]);
  }
  if (nthreads > 1)
    for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
}

/* ---- reduce-scatter (fp32 accumulation in rank order, one rounding) ---- */

static float ld_elem(const uint8_t* p, int dtype, int64_t e) {
  if (dtype == ORA_F32) {
    float f;
    memcpy(&f, p + 4 * e, 4);
    return f;
  }
  uint16_t h;
  memcpy(&h, p + 2 * e, 2);
  if (dtype == ORA_BF16) {
    uint32_t u = (uint32_t)h << 16;
    float f;
    memcpy(&f, &u, 4);
    return f;
  }
  _Float16 x;
  memcpy(&x, &h, 2);
  return (float)x;
}

static void st_elem(uint8_t* p, int dtype, int64_t e, float f) {
  if (dtype == ORA_F32) {
    memcpy(p + 4 * e, &f, 4);
    return;
  }
  uint16_t h;
  if (dtype == ORA_BF16) {
    uint32_t u;
    memcpy(&u, &f, 4);
    if ((u & 0x7f800000u) == 0x7f800000u && (u & 0x007fffffu)) h = (uint16_t)((u >> 16) | 0x40); /* quiet NaN */
    else h = (uint16_t)((u + 0x7fffu + ((u >> 16) & 1u)) >> 16);
  } else {
    _Float16 x = (_Float16)f; /* IEEE round to nearest even */
    memcpy(&h, &x, 2);
  }
  memcpy(p + 2 * e, &h, 2);
}

void ora_reduce_scatter(int dtype, int op, int64_t count, int n, uint8_t* const* in, uint8_t* const* out) {
  const int es = dtype == ORA_F32 ? 4 : 2;
  for (int j = 0; j < n; ++j)
    for (int64_t e = 0; e < count; ++e) {
      float acc = ld_elem(in[0] + (int64_t)j * count * es, dtype, e);
      for (int i = 1; i < n; ++i) {
        const float x = ld_elem(in[i] + (int64_t)j * count * es, dtype, e);
        if (op == ORA_SUM) acc = acc + x;
        else if (op == ORA_MAX) acc = (x > acc) ? x : acc;
        else acc = (x < acc) ? x : acc;
      }
      st_elem(out[j], dtype, e, acc);
    }
}
