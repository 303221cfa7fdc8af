// Plan lowering: a command program (program.hpp) or the SM path onto
// concrete buffers — lanes, flag operations, item / reduction tables and the
// prelaunch graphs.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <map>
#include <set>
#include <stdexcept>

#include "internal.hpp"

namespace cecoll {

namespace {

struct Addressing {
  std::vector<const char*> send;  // per rank, usable in this process
  std::vector<char*> recv;
};

// Address of `mine` (a pointer of local rank `me`) in rank `target`'s
// registered window at the same offset. The latest registration covering the
// pointer wins (an older window over the same allocator block may still be
// listed).
char* translate(World* w, int me, int target, const void* mine, bool* ok) {
  const char* p = static_cast<const char*>(mine);
  for (auto it = w->windows.rbegin(); it != w->windows.rend(); ++it) {
    const Window& win = *it;
    if (!win.live) continue;
    const char* b = win.rank_base[me];
    if (b && p >= b && p < b + win.bytes && win.rank_base[target]) return win.rank_base[target] + (p - b);
  }
  *ok = false;
  return nullptr;
}

uint64_t* slot(World* w, int rank, int index) { return w->flag_page[rank] + index; }

Item make_item(ItemKind kind, const char* src, char* dst, char* dst2, int64_t bytes) {
  Item it;
  std::memset(&it, 0, sizeof(it));
  it.kind = kind;
  it.src = src;
  it.dst = dst;
  it.dst2 = dst2;
  it.bytes = bytes;
  return it;
}

// A host-side item plus, for kItemFan, its destination list. `remote`: some
// destination is another device's memory (NVLink); such tables use the
// register mover (plain st.global to peer-mapped addresses) rather than TMA
// bulk stores.
struct HostItem {
  Item item;
  std::vector<char*> fan;
  bool remote = false;
};

// Chooses the mover (TMA for aligned copy/fan tables unless
// CECOLL_MOVER=reg), numbers the tiles, uploads the fan lists and the table.
Status upload_items(Plan* p, int device, std::vector<HostItem>& host, ItemTable* out) {
  if (host.empty()) return {};
  if (host.size() > static_cast<size_t>(kMaxItemsSmem))
    return fail(CECOLL_INVALID_ARGUMENT, "too many chunk transfers for one launch");
  DeviceGuard g(device);
  bool tma = true;
  // CECOLL_PEER_TMA=1 (read per plan): TMA bulk stores into peer-device
  // memory too (measured only on a multi-GPU node; default: register mover).
  const char* pt = std::getenv("CECOLL_PEER_TMA");
  const bool peer_tma = pt && std::string(pt) == "1";
  int kinds = 0;
  size_t nfan = 0;
  for (const HostItem& h : host) {
    const Item& it = h.item;
    kinds |= 1 << it.kind;
    uintptr_t a = reinterpret_cast<uintptr_t>(it.src) | reinterpret_cast<uintptr_t>(it.dst);
    for (char* f : h.fan) a |= reinterpret_cast<uintptr_t>(f);
    tma &= (it.kind == kItemCopy || it.kind == kItemFan || it.kind == kItemSwap) && (a & 15) == 0 &&
           (it.bytes & 15) == 0 && (!h.remote || peer_tma);
    nfan += h.fan.size();
  }
  // Swap items take the TMA mover only as a pure swap table (a stage holds
  // both sides of the exchange); CECOLL_TMA_SWAP=0 keeps them on registers.
  const char* ts = std::getenv("CECOLL_TMA_SWAP");
  if ((kinds & (1 << kItemSwap)) && (kinds != (1 << kItemSwap) || (ts && std::string(ts) == "0"))) tma = false;
  const char* env = std::getenv("CECOLL_MOVER");
  if (env && std::string(env) == "reg") tma = false;
  out->mover = tma ? Mover::Tma : Mover::Reg;
  out->kinds = kinds;
  char** fan_dev = nullptr;
  if (nfan) {
    std::vector<char*> flat;
    for (const HostItem& h : host) flat.insert(flat.end(), h.fan.begin(), h.fan.end());
    void* d = nullptr;
    CUDA_TRY(cudaMalloc(&d, sizeof(char*) * flat.size()));
    STATUS_TRY(write_device(d, flat.data(), sizeof(char*) * flat.size()));
    p->dev_allocs.push_back(d);
    p->dev_alloc_device.push_back(device);
    fan_dev = static_cast<char**>(d);
  }
  std::vector<int64_t> sizes;
  for (const HostItem& h : host) sizes.push_back(h.item.bytes);
  out->tile = table_tile(out->mover, sizes, p->sms, p->sm_budget, (kinds & (1 << kItemFan)) != 0,
                         kinds == (1 << kItemSwap));
  std::vector<Item> items;
  int64_t tiles = 0;
  size_t fan_at = 0;
  for (HostItem& h : host) {
    Item it = h.item;
    it.first_tile = static_cast<int32_t>(tiles);
    tiles += tiles_of(it.bytes, out->tile);
    if (it.kind == kItemFan) {
      it.fan = fan_dev + fan_at;
      it.nfan = static_cast<int32_t>(h.fan.size());
      it.dst = h.fan[0];
      fan_at += h.fan.size();
    }
    items.push_back(it);
  }
  if (tiles > INT32_MAX) return fail(CECOLL_INVALID_ARGUMENT, "collective too large for one launch");
  void* d = nullptr;
  CUDA_TRY(cudaMalloc(&d, sizeof(Item) * items.size()));
  STATUS_TRY(write_device(d, items.data(), sizeof(Item) * items.size()));
  p->dev_allocs.push_back(d);
  p->dev_alloc_device.push_back(device);
  out->items = static_cast<Item*>(d);
  out->nitems = static_cast<int>(items.size());
  out->ntiles = static_cast<int>(tiles);
  const int64_t per = tiles_of(items[0].bytes, out->tile);
  bool uniform = per > 0;
  for (const Item& it : items) uniform &= tiles_of(it.bytes, out->tile) == per;
  out->uniform = uniform ? static_cast<int>(per) : 0;
  return {};
}

Status upload_ptrs(Plan* p, int device, const std::vector<uint64_t*>& ptrs, uint64_t*** out) {
  *out = nullptr;
  if (ptrs.empty()) return {};
  DeviceGuard g(device);
  void* d = nullptr;
  CUDA_TRY(cudaMalloc(&d, sizeof(uint64_t*) * ptrs.size()));
  STATUS_TRY(write_device(d, ptrs.data(), sizeof(uint64_t*) * ptrs.size()));
  p->dev_allocs.push_back(d);
  p->dev_alloc_device.push_back(device);
  *out = static_cast<uint64_t**>(d);
  return {};
}

struct PlanReleaser {
  World* w;
  void operator()(Plan* p) const {
    plan_destroy(w, p);
    delete p;
  }
};

// Device holding the flag page that contains addr (-1 if none).
int flag_device(World* w, const uint64_t* addr) {
  for (int r = 0; r < w->nranks; ++r) {
    const uint64_t* b = w->flag_page[r];
    if (b && addr >= b && addr < b + kFlagBytes / sizeof(uint64_t)) return w->device[r];
  }
  return -1;
}

// Moves the writes in `ops` that target another device's flag page into
// `remote`: those are issued by a signal kernel (st.release.sys to the
// peer-mapped page) rather than a stream memory operation, the portable way
// to signal across NVLink. Same-device pages (also across processes) keep
// the memop.
void split_writes(World* w, int device, MemOps& ops, std::vector<uint64_t*>& remote, bool force) {
  MemOps keep;
  for (const auto& op : ops) {
    if (op.operation == CU_STREAM_MEM_OP_WRITE_VALUE_64) {
      uint64_t* a = reinterpret_cast<uint64_t*>(op.writeValue.address);
      const int d = flag_device(w, a);
      if (force || (d >= 0 && d != device)) {
        remote.push_back(a);
        continue;
      }
    }
    keep.push_back(op);
  }
  ops.swap(keep);
}

Status split_remote(World* w, Plan* p) {
  // CECOLL_REMOTE_SIGNAL=memop (read per plan): peer-device flags are written
  // by stream memory operations too, so the copy-engine path launches no
  // kernel at all (measured only on a multi-GPU node; default: signal kernel).
  const char* rs = std::getenv("CECOLL_REMOTE_SIGNAL");
  if (rs && std::string(rs) == "memop") return {};
  // CECOLL_FORCE_REMOTE_SIGNALS=1 (read per plan; tests): every cross-unit
  // signal takes the other-device path, so one GPU exercises it.
  const char* fr = std::getenv("CECOLL_FORCE_REMOTE_SIGNALS");
  const bool force = fr && std::string(fr) == "1";
  for (Unit& u : p->units) {
    split_writes(w, u.device, u.start, u.start_remote, force);
    split_writes(w, u.device, u.sm_post, u.sm_post_remote, force);
    STATUS_TRY(upload_ptrs(p, u.device, u.start_remote, &u.start_remote_tab));
    STATUS_TRY(upload_ptrs(p, u.device, u.sm_post_remote, &u.sm_post_remote_tab));
  }
  for (LaneExec& l : p->lanes) {
    const int dev = w->device[l.rank];
    std::vector<uint64_t*> remote;
    split_writes(w, dev, l.post, remote, force);
    for (Unit& u : p->units)
      if (std::find(u.ranks.begin(), u.ranks.end(), l.rank) != u.ranks.end())
        u.lanes_remote.insert(u.lanes_remote.end(), remote.begin(), remote.end());
  }
  for (Unit& u : p->units) STATUS_TRY(upload_ptrs(p, u.device, u.lanes_remote, &u.lanes_remote_tab));
  return {};
}


// Zeroed device words for a fused kernel: [0] err (u64), [1] ticket counter.
Status alloc_fused_words(Plan* p, int device, uint64_t** err, unsigned** ctr) {
  DeviceGuard g(device);
  void* d = nullptr;
  CUDA_TRY(cudaMalloc(&d, 64));
  STATUS_TRY(write_device(d, nullptr, 64));
  p->dev_allocs.push_back(d);
  p->dev_alloc_device.push_back(device);
  *err = static_cast<uint64_t*>(d);
  *ctr = reinterpret_cast<unsigned*>(static_cast<uint64_t*>(d) + 1);
  return {};
}

bool fusion_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("CECOLL_FUSED");
    return !(e && std::string(e) == "0");
  }();
  return on;
}

// SM path: the unit's rdy polls and done signals move into its item kernel.
Status fuse_sm_flags(World* w, Plan* p) {
  if (!fusion_enabled() || p->hybrid) return {};  // hybrid: lanes need the rdy polls too
  // When no rank outside a unit lives on its device (one process per GPU,
  // or one unit per device in a single process) the unit's start signals
  // fold into its kernel too: no other unit's kernel on this device can be
  // starved by the spinning grid, so writing them at kernel start is as good
  // as a separate submission ahead of it. The count is over every rank of the
  // world (w->device), not only this process's units: ranks of other
  // processes sharing the GPU (co-resident processes, MPS) have kernels that
  // our grid could starve.
  std::map<int, int> ranks_on;
  for (int r = 0; r < w->nranks; ++r) ++ranks_on[w->device[r]];
  for (Unit& u : p->units) {
    const bool distinct = ranks_on[u.device] == static_cast<int>(u.ranks.size());
    if (!u.table.nitems && !u.red.nitems) continue;  // the mover or the reduction carries them
    std::vector<uint64_t*> polls, sigs;
    for (const auto& op : u.sm_pre)
      if (op.operation == CU_STREAM_MEM_OP_WAIT_VALUE_64) polls.push_back(reinterpret_cast<uint64_t*>(op.waitValue.address));
    for (const auto& op : u.sm_post) sigs.push_back(reinterpret_cast<uint64_t*>(op.writeValue.address));
    sigs.insert(sigs.end(), u.sm_post_remote.begin(), u.sm_post_remote.end());
    if (polls.empty() && sigs.empty()) continue;  // nothing to fuse: plain kernel
    std::vector<uint64_t*> pre;
    if (distinct) {
      for (const auto& op : u.start) pre.push_back(reinterpret_cast<uint64_t*>(op.writeValue.address));
      pre.insert(pre.end(), u.start_remote.begin(), u.start_remote.end());
    }
    uint64_t** pt = nullptr;
    uint64_t** st = nullptr;
    uint64_t** prt = nullptr;
    STATUS_TRY(upload_ptrs(p, u.device, polls, &pt));
    STATUS_TRY(upload_ptrs(p, u.device, sigs, &st));
    STATUS_TRY(upload_ptrs(p, u.device, pre, &prt));
    u.sm_flags.pre = prt;
    u.sm_flags.npre = static_cast<int>(pre.size());
    u.start_folded = !pre.empty();
    u.sm_flags.polls = pt;
    u.sm_flags.npoll = static_cast<int>(polls.size());
    u.sm_flags.sigs = st;
    u.sm_flags.nsig = static_cast<int>(sigs.size());
    STATUS_TRY(alloc_fused_words(p, u.device, &u.sm_flags.err, &u.sm_flags.ctr));
    u.err = u.sm_flags.err;  // plan_destroy reports poll timeouts from here
    u.fused = true;
  }
  return {};
}

}  // namespace


namespace {

void set_key(Plan* p, const std::vector<CallArgs>& args) {
  for (const CallArgs& a : args) {
    p->key_rank.push_back(a.rank);
    p->key_send.push_back(a.send);
    p->key_recv.push_back(a.recv);
    p->key_stream.push_back(a.stream);
  }
}

// Every rank's send (and recv) as usable from this process: the call's own
// pointers for local ranks, the peers' through the registered windows.
Status resolve_addresses(World* w, const std::vector<CallArgs>& args, bool with_recv, Addressing* ad) {
  const int n = w->nranks;
  ad->send.assign(n, nullptr);
  ad->recv.assign(n, nullptr);
  std::vector<bool> have(n, false);
  for (const CallArgs& a : args) {
    if (a.rank < 0 || a.rank >= n || !w->local[a.rank]) return fail(CECOLL_INVALID_ARGUMENT, "rank not local");
    if (have[a.rank]) return fail(CECOLL_INVALID_ARGUMENT, "rank appears twice in one group");
    have[a.rank] = true;
    ad->send[a.rank] = static_cast<const char*>(a.send);
    ad->recv[a.rank] = static_cast<char*>(a.recv);
  }
  if (!w->multiprocess) {
    for (int r = 0; r < n; ++r)
      if (!have[r])
        return fail(CECOLL_INVALID_ARGUMENT,
                    "single-process communicator: every rank must take part (use cecoll_group_start/end)");
    return {};
  }
  if (static_cast<int>(args.size()) != w->nlocal)
    return fail(CECOLL_INVALID_ARGUMENT, "multi-process: every local rank must take part (group calls)");
  const CallArgs& a = args[0];
  for (int r = 0; r < n; ++r) {
    if (have[r]) continue;
    bool ok = true;
    ad->send[r] = translate(w, a.rank, r, a.send, &ok);
    if (with_recv) ad->recv[r] = translate(w, a.rank, r, a.recv, &ok);
    if (!ok)
      return fail(CECOLL_NOT_REGISTERED, with_recv ? "send/recv must lie in a window registered with cecoll_register"
                                                   : "send must lie in a window registered with cecoll_register");
  }
  return {};
}

// Units: the local ranks sharing (device, stream). Returns unit_of[rank]
// (-1 for ranks of other processes).
std::vector<int> form_units(World* w, Plan* p, const std::vector<CallArgs>& args) {
  std::vector<int> unit_of(w->nranks, -1);
  for (const CallArgs& a : args) {
    int found = -1;
    for (size_t u = 0; u < p->units.size(); ++u)
      if (p->units[u].device == w->device[a.rank] && p->units[u].stream == a.stream) found = static_cast<int>(u);
    if (found < 0) {
      Unit u;
      u.device = w->device[a.rank];
      u.stream = a.stream;
      p->units.push_back(u);
      found = static_cast<int>(p->units.size()) - 1;
    }
    p->units[found].ranks.push_back(a.rank);
    unit_of[a.rank] = found;
  }
  for (Unit& u : p->units) std::sort(u.ranks.begin(), u.ranks.end());
  return unit_of;
}

// Flag operations of the edges (r, j) between units: j
// announces (rdy[j] in r's page) and waits for done[r]; with `unit_level`
// (SM, hybrid, pull, reduce-scatter) r's unit polls rdy[j] and signals
// done[r] itself — otherwise r's lanes do (lower_program).
void add_edges(World* w, Plan* p, const std::vector<std::pair<int, int>>& edges, const std::vector<int>& unit_of,
               bool unit_level) {
  for (auto [r, j] : edges) {
    if (unit_of[r] >= 0 && unit_of[r] == unit_of[j]) continue;  // stream order suffices
    if (unit_of[j] >= 0) {
      Unit& u = p->units[unit_of[j]];
      u.start.push_back(op_write(slot(w, r, kSlotRdy + j), 1));
      add_poll(u.finish, slot(w, j, kSlotDone + r));
    }
    if (unit_of[r] >= 0 && unit_level) {
      Unit& u = p->units[unit_of[r]];
      add_poll(u.sm_pre, slot(w, r, kSlotRdy + j));
      u.sm_post.push_back(op_write(slot(w, j, kSlotDone + r), 1));
    }
  }
}

int device_sms(int device) {
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  return sms;
}

// Hybrid and pull. Each chunk: bytes [0, ce) by a
// copy-engine lane (lane d-1 of rank r carries the chunk to (r+d)%n, the
// pcpy rotation of compiler.cpp:150 — or, pulling, reads it from there),
// bytes [ce, s) by the unit's SM mover; the local slot entirely by the mover.
Status lower_hybrid(World* w, Plan* p, Kind kind, int64_t s, const Addressing& ad) {
  const int n = w->nranks;
  const int64_t sm_b = p->hybrid_sm_bytes, ce = s - sm_b;
  for (Unit& u : p->units) {
    std::vector<HostItem> items;
    for (int r : u.ranks) {
      const char* src_ag = ad.send[r];
      for (const Copy& c : u.placement)
        if (c.dst == ad.recv[r] + r * s) items.push_back({make_item(kItemCopy, c.src, c.dst, nullptr, c.bytes), {}});
      if (kind == Kind::AllGather && sm_b > 0) {
        HostItem h{make_item(kItemFan, src_ag + ce, nullptr, nullptr, sm_b), {}};
        for (int d = 1; d < n; ++d) {
          const int j = (r + d) % n;
          h.fan.push_back(ad.recv[j] + r * s + ce);
          h.remote |= w->device[j] != u.device;
        }
        if (h.fan.size() == 1) h.item = make_item(kItemCopy, src_ag + ce, h.fan[0], nullptr, sm_b), h.fan.clear();
        items.push_back(h);
      }
      for (int d = 1; d < n; ++d) {
        const int j = (r + d) % n;
        // push: r's chunk to j; pull: j's chunk read into r (lane d-1 of r either way)
        const char* src = p->pull ? (kind == Kind::AllGather ? ad.send[j] : ad.send[j] + r * s)
                                  : (kind == Kind::AllGather ? src_ag : ad.send[r] + j * s);
        char* dst = p->pull ? ad.recv[r] + j * s : ad.recv[j] + r * s;
        if (kind == Kind::AllToAll && sm_b > 0)
          items.push_back({make_item(kItemCopy, src + ce, dst + ce, nullptr, sm_b), {}, w->device[j] != u.device});
        if (ce > 0) {
          LaneExec le;
          le.rank = r;
          le.lane = d - 1;
          le.copies.push_back({dst, src, ce});
          STATUS_TRY(ensure_lanes(w->local[r].get(), d));
          p->lanes.push_back(std::move(le));
        }
      }
    }
    u.placement.clear();
    STATUS_TRY(upload_items(p, u.device, items, &u.table));
  }
  return {};
}

// The SM path: one item table per unit holding every chunk
// of its ranks, the local placement included.
Status lower_sm(World* w, Plan* p, Kind kind, int64_t s, const Addressing& ad) {
  const int n = w->nranks;
  for (Unit& u : p->units) {
    std::vector<HostItem> items;
    for (int r : u.ranks) {
      if (kind == Kind::AllGather) {
        // One read of the source chunk, one write per rank's slot r (local
        // slot first, then the pcpy rotation): n*s + n*n*s bytes instead of
        // 2*n*n*s for n separate copies.
        HostItem h{make_item(kItemFan, ad.send[r], nullptr, nullptr, s), {}};
        for (int d = 0; d < n; ++d) {
          char* dst = ad.recv[(r + d) % n] + r * s;
          if (dst != ad.send[r]) h.fan.push_back(dst);
          h.remote |= w->device[(r + d) % n] != u.device;
        }
        if (h.fan.size() == 1) h.item = make_item(kItemCopy, ad.send[r], h.fan[0], nullptr, s), h.fan.clear();
        if (!h.fan.empty() || h.item.kind == kItemCopy) items.push_back(h);
        continue;
      }
      for (const Copy& c : u.placement)
        if (c.dst == ad.recv[r] + r * s) items.push_back({make_item(kItemCopy, c.src, c.dst, nullptr, c.bytes), {}});
      for (int d = 1; d < n; ++d) {
        const int j = (r + d) % n;
        items.push_back({make_item(kItemCopy, ad.send[r] + j * s, ad.recv[j] + r * s, nullptr, s), {},
                         w->device[j] != u.device});
      }
    }
    u.placement.clear();
    STATUS_TRY(upload_items(p, u.device, items, &u.table));
  }
  return {};
}

// A command program's lanes: copies stay copy-engine
// commands; broadcast / swap become item kernels. A recorded (prelaunch)
// graph moves its same-device chunks with one item kernel per unit instead
// of one memcpy node per copy: the driver runs same-device memcpy on SMs
// anyway (profiles/ce_probe2_r01.txt) and every graph node costs launch
// latency. Cross-device copies stay memcpy nodes (copy engines over NVLink).
// CECOLL_GRAPH_MEMCPY=1 keeps every copy a memcpy node.
Status lower_program(World* w, Plan* p, const Addressing& ad, const std::vector<int>& unit_of, bool in_place_impl) {
  auto base = [&](int rank, Buf b) -> char* {  // in place (swap): Input is `recv` (compiler.cpp:119-122)
    if (in_place_impl || b == Buf::Output) return ad.recv[rank];
    return const_cast<char*>(ad.send[rank]);
  };
  auto addr = [&](const Region& r) { return base(r.rank, r.buf) + r.off; };
  auto same_unit = [&](int a, int b) { return unit_of[a] >= 0 && unit_of[a] == unit_of[b]; };
  const char* gm = std::getenv("CECOLL_GRAPH_MEMCPY");
  const bool merge = p->prelaunch && !(gm && std::string(gm) == "1");
  std::vector<std::vector<HostItem>> unit_items(p->units.size());
  if (merge)
    for (size_t ui = 0; ui < p->units.size(); ++ui) {
      for (const Copy& c : p->units[ui].placement)
        unit_items[ui].push_back({make_item(kItemCopy, c.src, c.dst, nullptr, c.bytes), {}});
      p->units[ui].placement.clear();
    }
  // Outside recorded prelaunch graphs, the broadcast / swap commands (item
  // kernels: no copy-engine form) of lanes that exchange no flags — every
  // destination in the same unit — also merge into the unit's one item
  // kernel, launched beside the lanes (exec.cpp run_ce): one kernel instead
  // of one per lane. Copies stay copy-engine commands. Below 4 MiB chunks
  // only: above, the lanes' concurrent kernels move broadcast / swap traffic
  // 7-10% faster (profiles/sweep_r01_plan_n8_merged.csv vs
  // sweep_r01_plan_n8_recorded.csv). CECOLL_MERGE_KERNELS=0 keeps one kernel
  // per lane; CECOLL_MERGE_KERNELS_MAX=<bytes> moves the cutoff.
  const char* mk = std::getenv("CECOLL_MERGE_KERNELS");
  const char* mkx = std::getenv("CECOLL_MERGE_KERNELS_MAX");
  const int64_t merge_max = mkx ? std::atoll(mkx) : (int64_t{4} << 20);
  const bool merge_kernels = !p->prelaunch && !(mk && std::string(mk) == "0") && p->chunk < merge_max;
  auto lane_dests = [&](const Lane& l) {
    std::set<int> d;
    for (const Command& c : l.cmds) {
      if (!c.moves_data()) continue;
      d.insert(c.op == Op::Swap ? c.peer.rank : c.dst.rank);
      if (c.op == Op::Broadcast) d.insert(c.dst2.rank);
    }
    d.erase(l.rank);
    return d;
  };
  for (const Lane& l : p->program.lanes) {  // lanes owned by local ranks
    if (unit_of[l.rank] < 0) continue;
    LaneExec le;
    le.rank = l.rank;
    le.lane = l.index;
    std::set<int> dests;
    std::vector<HostItem> items;
    const int dev = w->device[l.rank];
    bool flagless = true;
    for (int j : lane_dests(l)) flagless &= same_unit(l.rank, j);
    for (const Command& c : l.cmds) {
      const bool local_cmd = w->device[c.src.rank] == dev && w->device[c.dst.rank] == dev &&
                             (c.op != Op::Broadcast || w->device[c.dst2.rank] == dev) &&
                             (c.op != Op::Swap || w->device[c.peer.rank] == dev);
      const bool to_unit = local_cmd && (merge || (merge_kernels && flagless && c.op != Op::Copy));
      std::vector<HostItem>& sink = to_unit ? unit_items[unit_of[l.rank]] : items;
      switch (c.op) {
        case Op::Copy:
          if (merge && local_cmd) sink.push_back({make_item(kItemCopy, addr(c.src), addr(c.dst), nullptr, c.size), {}});
          else le.copies.push_back({addr(c.dst), addr(c.src), c.size});
          dests.insert(c.dst.rank);
          break;
        case Op::Broadcast:
          sink.push_back({make_item(kItemBcst, addr(c.src), addr(c.dst), addr(c.dst2), c.size), {}, !local_cmd});
          dests.insert(c.dst.rank);
          dests.insert(c.dst2.rank);
          break;
        case Op::Swap:
          sink.push_back({make_item(kItemSwap, addr(c.peer), addr(c.src), nullptr, c.size), {}, !local_cmd});
          dests.insert(c.peer.rank);
          break;
        default: break;  // Signal / Poll: realised by the flag operations below
      }
    }
    dests.erase(l.rank);
    for (int j : dests) {
      if (same_unit(l.rank, j)) continue;
      add_poll(le.pre, slot(w, l.rank, kSlotRdy + j));
      le.post.push_back(op_write(slot(w, j, kSlotDone + l.rank), 1));
    }
    STATUS_TRY(upload_items(p, w->device[l.rank], items, &le.table));
    STATUS_TRY(ensure_lanes(w->local[l.rank].get(), l.index + 1));
    p->lanes.push_back(std::move(le));
  }
  for (size_t ui = 0; ui < p->units.size(); ++ui)
    STATUS_TRY(upload_items(p, p->units[ui].device, unit_items[ui], &p->units[ui].table));
  return {};
}

}  // namespace

Impl select_for(World* w, Kind kind, int64_t s) {
  if (w->sm_budget == 0) {  // a budget changes the preference: the static policy decides
    const Impl t = tuned_select(w, kind, s);
    if (t != Impl::Auto) return t;
  }
  return select(kind, s, w->nranks, w->ndevices, w->sm_budget);
}

Status plan_create(World* w, Kind kind, Impl impl, int64_t s, const std::vector<CallArgs>& args, Plan** out,
                   const Program* given, bool no_placement) {
  const int n = w->nranks;
  if (s <= 0) return fail(CECOLL_INVALID_ARGUMENT, "collective: chunk size must be positive");
  // Frees device allocations, graphs and pinned pages if creation fails.
  std::unique_ptr<Plan, PlanReleaser> plan(new Plan, PlanReleaser{w});
  Plan* p = plan.get();
  p->kind = kind;
  p->chunk = s;
  set_key(p, args);
  if (given) {
    if (given->spec.kind != kind || given->spec.chunk != s || given->spec.nranks != n)
      return fail(CECOLL_INVALID_ARGUMENT, "program spec does not match the communicator / call");
    const std::string v = validate(*given, kMaxLanes);
    if (!v.empty()) return fail(CECOLL_INVALID_ARGUMENT, "program rejected: " + v);
    impl = given->impl;
  }
  if (impl == Impl::Auto) {
    bool in_place = kind == Kind::AllToAll;
    for (const CallArgs& a : args) in_place &= a.send == a.recv;
    impl = in_place ? Impl::Swap : select_for(w, kind, s);
  }
  if (impl != Impl::Sm && impl != Impl::Hybrid && impl != Impl::Pull && !valid_for(impl, kind))
    return fail(CECOLL_UNSUPPORTED, std::string(impl_name(impl)) + " does not apply to " +
                                         (kind == Kind::AllGather ? "allgather" : "alltoall"));
  const bool in_place_impl = base_of(impl) == Impl::Swap;
  p->impl = impl;
  p->sm_budget = w->sm_budget;
  // Pull runs on the hybrid executor with no SM share: the SM path's flag
  // edges (r, (r+d)%n) read as "reader r, source (r+d)%n" — the source's rdy
  // means "my send is ready", the reader's done "I have read it", exactly the
  // reduce-scatter's reader-side protocol; the reader's own recv is free by
  // its stream order.
  p->sm = impl == Impl::Sm || impl == Impl::Hybrid || impl == Impl::Pull;
  p->hybrid = impl == Impl::Hybrid || impl == Impl::Pull;
  p->pull = impl == Impl::Pull;
  p->prelaunch = is_prelaunched(impl);
  if (p->hybrid) {
    const char* e = std::getenv("CECOLL_HYBRID_SM_PCT");
    int pct = e ? std::atoi(e) : 50;
    pct = std::max(0, std::min(100, pct));
    p->hybrid_sm_bytes = p->pull ? 0 : (s * pct / 100) & ~int64_t{15};
  }

  Addressing ad;
  STATUS_TRY(resolve_addresses(w, args, true, &ad));
  for (const CallArgs& a : args)
    if (kind == Kind::AllToAll && a.send == a.recv && !in_place_impl)
      return fail(CECOLL_INVALID_ARGUMENT, "alltoall in place requires the swap implementation");
  const std::vector<int> unit_of = form_units(w, p, args);

  // Edges writer -> destination (SM / hybrid: every pair; pull: reader ->
  // source) and the flag operations they imply.
  std::vector<std::pair<int, int>> edges;
  if (p->sm) {
    for (int r = 0; r < n; ++r)
      for (int d = 1; d < n; ++d) edges.push_back({r, (r + d) % n});
  } else {
    if (n < 2) return fail(CECOLL_INVALID_ARGUMENT, "collective: gpu_count must be >= 2");
    Spec spec;
    spec.kind = kind;
    spec.chunk = s;
    spec.nranks = n;
    try {
      p->program = given ? *given : compile(impl, spec, kMaxLanes);
    } catch (const std::invalid_argument& e) {
      return fail(CECOLL_INVALID_ARGUMENT, e.what());
    }
    for (const Lane& l : p->program.lanes)
      for (const Command& c : l.cmds) {
        if (!c.moves_data()) continue;
        const Region* ds[3] = {&c.dst, c.op == Op::Broadcast ? &c.dst2 : nullptr, nullptr};
        if (c.op == Op::Swap) ds[0] = &c.peer;
        for (const Region* d : ds)
          if (d && d->rank != l.rank) edges.push_back({l.rank, d->rank});
      }
  }
  add_edges(w, p, edges, unit_of, p->sm);

  // Local-slot placement (verifier.cpp:40-44) and the swap pre-copy.
  for (Unit& u : p->units)
    for (int r : u.ranks) {
      if (in_place_impl) {
        if (ad.send[r] != ad.recv[r]) u.precopy.push_back({ad.recv[r], ad.send[r], s * n});
        continue;
      }
      const char* src = ad.send[r] + (kind == Kind::AllGather ? 0 : r * s);
      char* dst = ad.recv[r] + r * s;
      if (src != dst && !no_placement) u.placement.push_back({dst, src, s});
    }

  p->sms = device_sms(p->units[0].device);  // tile sizes depend on it (upload_items)
  if (p->hybrid) STATUS_TRY(lower_hybrid(w, p, kind, s, ad));
  else if (p->sm) STATUS_TRY(lower_sm(w, p, kind, s, ad));
  else STATUS_TRY(lower_program(w, p, ad, unit_of, in_place_impl));
  STATUS_TRY(split_remote(w, p));
  if (p->sm) STATUS_TRY(fuse_sm_flags(w, p));
  if (p->prelaunch)
    for (Unit& u : p->units) {
      const Status gs = build_graph(w, p, u);
      if (gs.ok()) continue;
      if (given) return gs;  // a given program keeps its polls: no eager form
      // A graph this driver cannot record or instantiate (e.g. a copy-engine
      // memcpy node between devices inside a conditional body): run the same
      // command program without prelaunch rather than fail the collective.
      std::string why = gs.msg;
      Plan* eager = nullptr;  // `plan` (the failed one) is released on return
      STATUS_TRY(plan_create(w, kind, base_of(impl), s, args, &eager, given));
      eager->impl = impl;
      eager->graph_fallback = why;
      *out = eager;
      return {};
    }
  *out = plan.release();
  return {};
}

namespace {

// Uploads a reduction table: the items plus one flat array of source pointers.
Status upload_red(Plan* p, int device, std::vector<RedItem>& items, const std::vector<std::vector<const char*>>& srcs,
                  int dtype, int op, RedTable* out) {
  if (items.empty()) return {};
  if (items.size() > static_cast<size_t>(kMaxItemsSmem))
    return fail(CECOLL_INVALID_ARGUMENT, "too many reductions for one launch");
  DeviceGuard g(device);
  std::vector<const char*> flat;
  for (const auto& v : srcs) flat.insert(flat.end(), v.begin(), v.end());
  void* d = nullptr;
  CUDA_TRY(cudaMalloc(&d, sizeof(char*) * flat.size()));
  STATUS_TRY(write_device(d, flat.data(), sizeof(char*) * flat.size()));
  p->dev_allocs.push_back(d);
  p->dev_alloc_device.push_back(device);
  int64_t tiles = 0;
  size_t at = 0;
  for (size_t i = 0; i < items.size(); ++i) {
    items[i].srcs = static_cast<const char* const*>(d) + at;
    at += srcs[i].size();
    items[i].first_tile = static_cast<int32_t>(tiles);
    tiles += (items[i].elems + kRedTileElems - 1) / kRedTileElems;
  }
  if (tiles > INT32_MAX) return fail(CECOLL_INVALID_ARGUMENT, "reduce-scatter too large for one launch");
  void* t = nullptr;
  CUDA_TRY(cudaMalloc(&t, sizeof(RedItem) * items.size()));
  STATUS_TRY(write_device(t, items.data(), sizeof(RedItem) * items.size()));
  p->dev_allocs.push_back(t);
  p->dev_alloc_device.push_back(device);
  out->items = static_cast<RedItem*>(t);
  out->nitems = static_cast<int>(items.size());
  out->ntiles = static_cast<int>(tiles);
  out->dtype = dtype;
  out->op = op;
  return {};
}

RedItem make_red(char* dst, int64_t elems, const std::vector<const char*>& srcs, int esize) {
  RedItem r;
  std::memset(&r, 0, sizeof(r));
  r.dst = dst;
  r.elems = elems;
  r.nsrc = static_cast<int32_t>(srcs.size());
  uintptr_t a = reinterpret_cast<uintptr_t>(dst);
  for (const char* s : srcs) a |= reinterpret_cast<uintptr_t>(s);
  r.vec = (a & 15) == 0 && esize > 0;
  return r;
}

}  // namespace

Status plan_create_rs(World* w, Impl impl, int64_t count, int dtype, int op, const std::vector<CallArgs>& args,
                      Plan** out) {
  const int n = w->nranks;
  if (count <= 0) return fail(CECOLL_INVALID_ARGUMENT, "reduce-scatter: count must be positive");
  if (dtype < kF32 || dtype > kF16 || op < kSum || op > kMin)
    return fail(CECOLL_INVALID_ARGUMENT, "reduce-scatter: unknown dtype or op");
  if (impl == Impl::Auto) impl = Impl::Sm;
  if (impl != Impl::Sm && impl != Impl::Pcpy && impl != Impl::B2b && impl != Impl::PrelaunchPcpy &&
      impl != Impl::PrelaunchB2b)
    return fail(CECOLL_UNSUPPORTED, "reduce-scatter: sm, pcpy, b2b, prelaunch_pcpy or prelaunch_b2b");
  const int esize = dtype_bytes(dtype);
  const int64_t s = count * esize;
  // Frees device allocations, graphs and pinned pages if creation fails.
  std::unique_ptr<Plan, PlanReleaser> plan(new Plan, PlanReleaser{w});
  Plan* p = plan.get();
  p->kind = Kind::ReduceScatter;
  p->impl = impl;
  p->chunk = s;
  p->dtype = dtype;
  p->op = op;
  p->sm = impl == Impl::Sm;
  p->sm_budget = w->sm_budget;
  set_key(p, args);
  if (w->multiprocess && !p->sm)
    return fail(CECOLL_UNSUPPORTED, "reduce-scatter over copy engines needs a single-process communicator");
  Addressing ad;  // the readers need every rank's send; recv stays local
  STATUS_TRY(resolve_addresses(w, args, false, &ad));
  const std::vector<const char*>& send = ad.send;
  const std::vector<char*>& recv = ad.recv;
  p->sms = device_sms(w->device[args[0].rank]);

  if (!p->sm) {
    // Copy-engine gather: chunk j of every rank lands in rank j's staging
    // slot i (an all-to-all into staging), then rank j reduces its staging.
    std::vector<CallArgs> inner_args;
    std::vector<char*> staging(n, nullptr);
    for (const CallArgs& a : args) {
      DeviceGuard g(w->device[a.rank]);
      void* d = nullptr;
      CUDA_TRY(cudaMalloc(&d, static_cast<size_t>(s) * n));
      p->dev_allocs.push_back(d);
      p->dev_alloc_device.push_back(w->device[a.rank]);
      staging[a.rank] = static_cast<char*>(d);
      inner_args.push_back({a.rank, a.send, d, a.stream});
    }
    // The gather skips each rank's own chunk (no local placement): the
    // reduction reads it in place, 2n·s fewer HBM bytes of (3n² + n)·s.
    Plan* inner = nullptr;
    STATUS_TRY(plan_create(w, Kind::AllToAll, impl, s, inner_args, &inner, nullptr, true));
    p->inner.reset(inner);
    for (const Unit& iu : inner->units) {
      Unit u;
      u.device = iu.device;
      u.stream = iu.stream;
      u.ranks = iu.ranks;
      std::vector<RedItem> items;
      std::vector<std::vector<const char*>> srcs;
      for (int j : u.ranks) {
        std::vector<const char*> v;
        for (int i = 0; i < n; ++i) v.push_back(i == j ? send[j] + j * s : staging[j] + i * s);
        items.push_back(make_red(recv[j], count, v, esize));
        srcs.push_back(v);
      }
      STATUS_TRY(upload_red(p, u.device, items, srcs, dtype, op, &u.red));
      p->units.push_back(std::move(u));
    }
    *out = plan.release();
    return {};
  }

  // SM path: units, flags (edge (r, j): rank r reads rank j's send), reductions.
  const std::vector<int> unit_of = form_units(w, p, args);
  std::vector<std::pair<int, int>> edges;
  for (int r = 0; r < n; ++r)
    for (int d = 1; d < n; ++d) edges.push_back({r, (r + d) % n});
  add_edges(w, p, edges, unit_of, true);
  for (Unit& u : p->units) {
    std::vector<RedItem> items;
    std::vector<std::vector<const char*>> srcs;
    for (int j : u.ranks) {
      std::vector<const char*> v;
      for (int i = 0; i < n; ++i) v.push_back(send[i] + j * s);
      items.push_back(make_red(recv[j], count, v, esize));
      srcs.push_back(v);
    }
    STATUS_TRY(upload_red(p, u.device, items, srcs, dtype, op, &u.red));
  }
  STATUS_TRY(split_remote(w, p));
  STATUS_TRY(fuse_sm_flags(w, p));
  *out = plan.release();
  return {};
}

namespace {

// Folded prelaunch body: the unit's mover kernel is its own
// gate. It spins from the moment it is armed, so it must leave the device to
// everything else: only small collectives fold (at most
// CECOLL_FOLD_MAX_TILES_PER_CTA tiles per CTA) and the grid is capped at
// CECOLL_FOLD_MAX_CTAS CTAs (default 32) split between the plan's units on the
// device, within the plan's SM budget. Returns the grid, or 0 for no fold.
int fold_grid(World* w, const Plan* p, const Unit& u) {
  static const int max_ctas = [] {
    const char* e = std::getenv("CECOLL_FOLD_MAX_CTAS");
    return e ? std::atoi(e) : 32;
  }();
  static const int max_tiles = [] {
    const char* e = std::getenv("CECOLL_FOLD_MAX_TILES_PER_CTA");
    return e ? std::atoi(e) : 4;
  }();
  // Off by default: measured slower than gate_poll -> mover on one B200
  // (profiles/prelaunch_fold_ab_r02.csv); CECOLL_PRELAUNCH_FOLD=1 enables.
  const char* on = std::getenv("CECOLL_PRELAUNCH_FOLD");
  if (!(on && std::string(on) == "1") || max_ctas <= 0) return 0;
  int units_here = 0;
  for (const Unit& v : p->units) units_here += v.device == u.device;
  (void)w;
  int cap = std::max(1, max_ctas / std::max(1, units_here));
  if (p->sm_budget > 0) cap = std::min(cap, p->sm_budget);
  const int grid = std::min(cap, u.table.ntiles);
  if (grid <= 0 || static_cast<int64_t>(grid) * max_tiles < u.table.ntiles) return 0;
  return grid;
}

}  // namespace

// Builds one unit's prelaunch graph explicitly (no stream capture; GraphSink):
//  * kernel-only body, folded: one mover kernel that takes the trigger word
//    itself (FlagSet::fold) — one kernel per collective;
//  * kernel-only body: gate_poll kernel -> mover (done signals fused);
//  * otherwise: gate kernel -> IF{ poll kernel -> lanes (memcpy nodes, item
//    kernels) + placement -> signal kernel }.
// Every form is triggered by the unit's trigger word (its ready slot), which
// the caller stream writes; no host memory is read on the trigger path.
Status build_graph(World* w, Plan* p, Unit& u) {
  DeviceGuard g(u.device);
  CUDA_TRY(cudaStreamCreateWithFlags(&u.arm, cudaStreamNonBlocking));
  CUDA_TRY(cudaEventCreateWithFlags(&u.graph_done, cudaEventDisableTiming));
  void* d = nullptr;
  CUDA_TRY(cudaMalloc(&d, 64));
  STATUS_TRY(write_device(d, nullptr, 64));
  p->dev_allocs.push_back(d);
  p->dev_alloc_device.push_back(u.device);
  uint64_t* words = static_cast<uint64_t*>(d);  // [0] trigger [1] err [2] ticket [3] skip [4] gate [5] epoch [6] seen
  u.err = words + 1;
  u.ready_flag = words;
  STATUS_TRY(upload_ptrs(p, u.device, {u.ready_flag}, &u.ready_tab));
  void* host = nullptr;
  CUDA_TRY(cudaHostAlloc(&host, 64, cudaHostAllocMapped | cudaHostAllocPortable));
  std::memset(host, 0, 64);
  u.cancel_host = static_cast<uint64_t*>(host);
  CUDA_TRY(cudaHostGetDevicePointer(reinterpret_cast<void**>(&u.cancel_dev), host, 0));
  uint64_t* const seen = words + 6;

  // Polls: the unit's trigger word first (the gate takes it), then rdy from
  // destinations in other units; signals: done to those destinations (from
  // the lanes' memops).
  std::vector<uint64_t*> polls{u.ready_flag}, sigs, fins;
  for (const LaneExec& le : p->lanes) {
    if (std::find(u.ranks.begin(), u.ranks.end(), le.rank) == u.ranks.end()) continue;
    for (const auto& op : le.pre)
      if (op.operation == CU_STREAM_MEM_OP_WAIT_VALUE_64) polls.push_back(reinterpret_cast<uint64_t*>(op.waitValue.address));
    for (const auto& op : le.post) sigs.push_back(reinterpret_cast<uint64_t*>(op.writeValue.address));
  }
  sigs.insert(sigs.end(), u.lanes_remote.begin(), u.lanes_remote.end());
  for (const auto& op : u.finish)
    if (op.operation == CU_STREAM_MEM_OP_WAIT_VALUE_64) fins.push_back(reinterpret_cast<uint64_t*>(op.waitValue.address));
  u.npoll = static_cast<int>(polls.size());
  u.nsig = static_cast<int>(sigs.size());
  u.nfin = static_cast<int>(fins.size());
  STATUS_TRY(upload_ptrs(p, u.device, polls, &u.poll_tab));
  STATUS_TRY(upload_ptrs(p, u.device, sigs, &u.sig_tab));
  STATUS_TRY(upload_ptrs(p, u.device, fins, &u.fin_tab));

  // Building the graph counts its commands in the world's counters; nothing
  // is submitted, so they are restored afterwards.
  int64_t before[kNumCounters];
  for (int i = 0; i < kNumCounters; ++i) before[i] = w->counters[i];
  struct Restore {
    World* w;
    int64_t* b;
    ~Restore() {
      for (int i = 0; i < kNumCounters; ++i) w->counters[i] = b[i];
    }
  } restore{w, before};

  // Kernel-only body (every chunk of the unit in its item kernel: no
  // copy-engine lanes, no placement copies): no conditional node.
  // CECOLL_PRELAUNCH_COND=1 keeps the conditional form for comparison.
  bool lanes_idle = u.placement.empty();
  for (const LaneExec& l : p->lanes)
    if (std::find(u.ranks.begin(), u.ranks.end(), l.rank) != u.ranks.end() && (!l.copies.empty() || l.table.nitems))
      lanes_idle = false;
  const char* pc = std::getenv("CECOLL_PRELAUNCH_COND");
  if (lanes_idle && u.table.nitems > 0 && fusion_enabled() && !(pc && std::string(pc) == "1")) {
    CUDA_TRY(cudaGraphCreate(&u.graph, 0));
    GraphSink sink({u.graph});
    FlagSet f;
    f.sigs = u.sig_tab;
    f.nsig = u.nsig;
    f.err = u.err;
    const int fg = fold_grid(w, p, u);
    if (fg > 0) {
      // One kernel: gate (trigger word), polls (rdy), move, signals; its
      // last CTA advances the instance count the next instance gates on.
      f.epoch = words + 5;
      f.cancel = u.cancel_dev;
      f.seen = seen;
      f.gate = words + 4;
      f.polls = u.poll_tab;
      f.npoll = u.npoll;
      f.ctr = reinterpret_cast<unsigned*>(words + 2);
      p->folded = true;
      STATUS_TRY(sink.kernel(w, u.arm, items_call(u.table, fg, &f)));
    } else {
      // The mover never spins here (gate_poll did the waiting), so it keeps a
      // full grid without holding SMs while armed.
      f.ctr = u.nsig ? reinterpret_cast<unsigned*>(words + 2) : nullptr;
      f.skip = words + 3;
      STATUS_TRY(sink.kernel(w, u.arm, gate_poll_call(u.poll_tab, u.npoll, u.cancel_dev, seen, words + 3, u.err)));
      STATUS_TRY(sink.kernel(w, u.arm, items_call(u.table, plan_grid(p, u.table), &f)));
      // CECOLL_PRELAUNCH_PDL=1: the gate -> mover edge becomes programmatic,
      // so the mover's CTAs launch while the gate finishes (tools/pdl_probe.cu)
      const char* pdl = std::getenv("CECOLL_PRELAUNCH_PDL");
      if (pdl && std::string(pdl) == "1") {
        size_t ne = 1;
        cudaGraphNode_t from = nullptr, to = nullptr;
        CUDA_TRY(cudaGraphGetEdges(u.graph, &from, &to, &ne));
        if (ne == 1) {
          CUDA_TRY(cudaGraphRemoveDependencies(u.graph, &from, &to, 1));
          cudaGraphEdgeData ed = {};
          ed.from_port = cudaGraphKernelNodePortProgrammatic;
          ed.type = cudaGraphDependencyTypeProgrammatic;
          CUDA_TRY(cudaGraphAddDependencies_v2(u.graph, &from, &to, &ed, 1));
        }
      }
    }
    CUDA_TRY(cudaGraphInstantiate(&u.exec, u.graph, 0));
    return {};
  }

  CUDA_TRY(cudaGraphCreate(&u.graph, 0));
  cudaGraphConditionalHandle handle;
  CUDA_TRY(cudaGraphConditionalHandleCreate(&handle, u.graph, 0, cudaGraphCondAssignDefault));
  GraphSink top({u.graph});
  STATUS_TRY(top.kernel(w, u.arm, gate_call(u.ready_flag, u.cancel_dev, seen, handle, u.err)));

  // cudaGraphNodeParams has no default constructor (union with non-trivial
  // members): zero-initialised raw storage, as the runtime expects.
  alignas(cudaGraphNodeParams) unsigned char cp_storage[sizeof(cudaGraphNodeParams)] = {};
  cudaGraphNodeParams& cp = *reinterpret_cast<cudaGraphNodeParams*>(cp_storage);
  cp.type = cudaGraphNodeTypeConditional;
  cp.conditional.handle = handle;
  cp.conditional.type = cudaGraphCondTypeIf;
  cp.conditional.size = 1;
  STATUS_TRY(top.add_node(u.arm, &cp, nullptr));
  cudaGraph_t body = cp.conditional.phGraph_out[0];

  // Body: poll -> fork lanes -> join -> signal. The body's waits stay in
  // one-CTA poll kernels: an armed instance runs ahead of the caller stream,
  // and a full-grid mover spinning on its flags could hold every SM that the
  // caller's own poll kernel (on which those flags transitively depend)
  // needs — measured as a deadlock with eight units on one GPU. Stream
  // memory operations are not allowed in conditional bodies, hence kernels.
  GraphSink sink({body});
  STATUS_TRY(sink.kernel(w, u.arm, poll_call(u.poll_tab + 1, u.npoll - 1, u.err)));  // [0]: the gate's
  STATUS_TRY(sink.copies(w, u.placement, u.arm));
  const cudaEvent_t fork = w->local[u.ranks[0]]->start;  // an ordering key inside the graph
  STATUS_TRY(sink.record(w, fork, u.arm));
  std::vector<const LaneExec*> busy;
  for (const LaneExec& l : p->lanes) {
    if (std::find(u.ranks.begin(), u.ranks.end(), l.rank) == u.ranks.end()) continue;
    if (l.copies.empty() && !l.table.nitems) continue;  // its chunks are in the unit kernel
    RankState* rs = w->local[l.rank].get();
    cudaStream_t ls = rs->lanes[l.lane];
    STATUS_TRY(sink.wait(w, ls, fork));
    STATUS_TRY(sink.copies(w, l.copies, ls));
    STATUS_TRY(sink.kernel(w, ls, items_call(l.table, plan_grid(p, l.table))));
    STATUS_TRY(sink.record(w, rs->lane_done[l.lane], ls));
    busy.push_back(&l);
  }
  // Same-device chunks of every lane of the unit: one item kernel.
  STATUS_TRY(sink.kernel(w, u.arm, items_call(u.table, plan_grid(p, u.table))));
  for (const LaneExec* l : busy) STATUS_TRY(sink.wait(w, u.arm, w->local[l->rank]->lane_done[l->lane]));
  STATUS_TRY(sink.kernel(w, u.arm, signal_call(u.sig_tab, u.nsig)));
  CUDA_TRY(cudaGraphInstantiate(&u.exec, u.graph, 0));
  return {};
}

}  // namespace cecoll
