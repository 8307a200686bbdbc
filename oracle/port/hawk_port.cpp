// TEST INFRASTRUCTURE ONLY — CPU restatement of the reference oracle for the
// five BASELINE queries (see hawk_port.h). Semantics cited per query:
//   comparisons            planner_reference.cpp:76-104
//   int64 wrap arithmetic  planner_reference.cpp:25-33, :129-136
//   unique-key inner join  planner_reference.cpp:164-187
//   SUM/COUNT/AVG          planner_reference.cpp:233-265, :305-308
//   empty non-grouped SUM  planner_reference.cpp:269-278 (one row, SUM = 0)
//
// Each query is one per-thread row body over the fact columns of a row range;
// port_run feeds it materialised columns, port_run_gen feeds it chunks that
// each worker regenerates from include/hawk_gen.h (the streaming oracle for
// SF100, where materialising the fact table on the host is not an option).
#include "hawk_port.h"

#include <algorithm>
#include <array>
#include <cstring>
#include <functional>
#include <map>
#include <thread>
#include <unordered_map>
#include <vector>

#include "hawk_gen.h"

namespace {

using u64 = uint64_t;

int64_t wadd(int64_t a, int64_t b) { return static_cast<int64_t>(static_cast<u64>(a) + static_cast<u64>(b)); }
int64_t wsub(int64_t a, int64_t b) { return static_cast<int64_t>(static_cast<u64>(a) - static_cast<u64>(b)); }
int64_t wmul(int64_t a, int64_t b) { return static_cast<int64_t>(static_cast<u64>(a) * static_cast<u64>(b)); }

int64_t dbits(double d) {
  int64_t b;
  std::memcpy(&b, &d, 8);
  return b;
}

template <typename F>
void parallel_for(int64_t n, int threads, F&& body) {
  threads = std::max(1, threads);
  if (threads == 1 || n < 4096) {
    body(0, int64_t{0}, n);
    return;
  }
  std::vector<std::thread> pool;
  const int64_t chunk = (n + threads - 1) / threads;
  for (int t = 0; t < threads; ++t) {
    const int64_t b = std::min(n, t * chunk), e = std::min(n, b + chunk);
    pool.emplace_back([&, t, b, e] { body(t, b, e); });
  }
  for (auto& th : pool) th.join();
}

// key -> row index for a dimension with non-negative unique keys
std::vector<int32_t> index_keys(const int64_t* keys, int64_t rows, const std::vector<bool>* keep) {
  int64_t mx = -1;
  for (int64_t i = 0; i < rows; ++i) mx = std::max(mx, keys[i]);
  std::vector<int32_t> idx(static_cast<std::size_t>(mx + 1), -1);
  for (int64_t i = 0; i < rows; ++i)
    if (!keep || (*keep)[static_cast<std::size_t>(i)]) idx[static_cast<std::size_t>(keys[i])] = static_cast<int32_t>(i);
  return idx;
}

int32_t lookup(const std::vector<int32_t>& idx, int64_t key) {
  return (key >= 0 && static_cast<std::size_t>(key) < idx.size()) ? idx[static_cast<std::size_t>(key)] : -1;
}

// generated columns of each query, in port_run's `cols` order (hawk_port.h)
struct ColRef {
  int table, col;
};
const std::vector<ColRef>& fact_columns(int q) {
  static const std::vector<ColRef> k[5] = {
      {{HG_LINEITEM, HG_L_SHIPDATE}, {HG_LINEITEM, HG_L_DISCOUNT}, {HG_LINEITEM, HG_L_QUANTITY},
       {HG_LINEITEM, HG_L_EXTENDEDPRICE}},
      {{HG_LINEITEM, HG_L_SHIPDATE}, {HG_LINEITEM, HG_L_RETURNFLAG}, {HG_LINEITEM, HG_L_LINESTATUS},
       {HG_LINEITEM, HG_L_QUANTITY}, {HG_LINEITEM, HG_L_EXTENDEDPRICE}, {HG_LINEITEM, HG_L_DISCOUNT},
       {HG_LINEITEM, HG_L_TAX}},
      {{HG_LINEORDER, HG_LO_ORDERDATE}, {HG_LINEORDER, HG_LO_DISCOUNT}, {HG_LINEORDER, HG_LO_QUANTITY},
       {HG_LINEORDER, HG_LO_EXTENDEDPRICE}},
      {{HG_LINEORDER, HG_LO_CUSTKEY}, {HG_LINEORDER, HG_LO_SUPPKEY}, {HG_LINEORDER, HG_LO_PARTKEY},
       {HG_LINEORDER, HG_LO_ORDERDATE}, {HG_LINEORDER, HG_LO_REVENUE}, {HG_LINEORDER, HG_LO_SUPPLYCOST}},
      {{HG_LINEITEM, HG_L_ORDERKEY}, {HG_LINEITEM, HG_L_SHIPDATE}, {HG_LINEITEM, HG_L_EXTENDEDPRICE},
       {HG_LINEITEM, HG_L_DISCOUNT}}};
  return k[q];
}
const std::vector<ColRef>& dim_columns(int q) {
  static const std::vector<ColRef> k[5] = {
      {},
      {},
      {{HG_DDATE, HG_D_DATEKEY}, {HG_DDATE, HG_D_YEAR}},
      {{HG_SCUSTOMER, HG_SC_CUSTKEY}, {HG_SCUSTOMER, HG_SC_REGION}, {HG_SCUSTOMER, HG_SC_NATION},
       {HG_SUPPLIER, HG_S_SUPPKEY}, {HG_SUPPLIER, HG_S_REGION}, {HG_PART, HG_P_PARTKEY},
       {HG_PART, HG_P_MFGR}, {HG_DDATE, HG_D_DATEKEY}, {HG_DDATE, HG_D_YEAR}},
      {{HG_ORDERS, HG_O_ORDERKEY}, {HG_ORDERS, HG_O_CUSTKEY}, {HG_ORDERS, HG_O_ORDERDATE},
       {HG_ORDERS, HG_O_SHIPPRIORITY}, {HG_CUSTOMER, HG_C_CUSTKEY}, {HG_CUSTOMER, HG_C_MKTSEGMENT}}};
  return k[q];
}
const std::vector<int>& dim_tables(int q) {
  static const std::vector<int> k[5] = {{}, {}, {HG_DDATE}, {HG_SCUSTOMER, HG_SUPPLIER, HG_PART, HG_DDATE},
                                        {HG_ORDERS, HG_CUSTOMER}};
  return k[q];
}

// Fact rows reach the query body as column pointers for a row range:
// feed(T, body) calls body(thread, fact_cols, rows) one or more times per
// thread, each call covering the next rows of the thread's range.
using Body = std::function<void(int, const int64_t* const*, int64_t)>;
using Feed = std::function<void(int, const Body&)>;

// The query bodies: per-thread state accumulates over the calls of a thread;
// c = dimension columns (index 0.. in dim_columns order), f = fact columns.
int64_t execute(int query, const int64_t* const* c, const int64_t* dim_rows, const int64_t* codes,
                int T, const Feed& feed, int64_t* out, int64_t out_rows) {
  switch (query) {
    case PORT_Q6: {
      // sum(l_extendedprice*l_discount) where l_shipdate >= 19940101 and
      // l_shipdate < 19950101 and l_discount >= 5 and l_discount <= 7 and l_quantity < 24
      std::vector<int64_t> part(static_cast<std::size_t>(T), 0);
      feed(T, [&](int t, const int64_t* const* f, int64_t n) {
        int64_t s = 0;
        for (int64_t i = 0; i < n; ++i)
          if (f[0][i] >= 19940101 && f[0][i] < 19950101 && f[1][i] >= 5 && f[1][i] <= 7 && f[2][i] < 24)
            s = wadd(s, wmul(f[3][i], f[1][i]));
        part[static_cast<std::size_t>(t)] = wadd(part[static_cast<std::size_t>(t)], s);
      });
      int64_t s = 0;
      for (int64_t p : part) s = wadd(s, p);
      if (out_rows < 1) return -1;
      out[0] = s;
      return 1;
    }
    case PORT_Q1: {
      // group by l_returnflag, l_linestatus where l_shipdate <= 19980902
      struct Acc { int64_t qty = 0, price = 0, disc_price = 0, charge = 0, disc = 0, count = 0; };
      using Map = std::map<std::pair<int64_t, int64_t>, Acc>;
      std::vector<Map> maps(static_cast<std::size_t>(T));
      feed(T, [&](int t, const int64_t* const* f, int64_t n) {
        Map& m = maps[static_cast<std::size_t>(t)];
        for (int64_t i = 0; i < n; ++i) {
          if (!(f[0][i] <= 19980902)) continue;
          Acc& a = m[{f[1][i], f[2][i]}];
          const int64_t q = f[3][i], ep = f[4][i], d = f[5][i], tx = f[6][i];
          const int64_t dp = wmul(ep, wsub(100, d));
          a.qty = wadd(a.qty, q);
          a.price = wadd(a.price, ep);
          a.disc_price = wadd(a.disc_price, dp);
          a.charge = wadd(a.charge, wmul(dp, wadd(100, tx)));
          a.disc = wadd(a.disc, d);
          ++a.count;
        }
      });
      Map all;
      for (const Map& m : maps)
        for (const auto& [k, a] : m) {
          Acc& x = all[k];
          x.qty = wadd(x.qty, a.qty);
          x.price = wadd(x.price, a.price);
          x.disc_price = wadd(x.disc_price, a.disc_price);
          x.charge = wadd(x.charge, a.charge);
          x.disc = wadd(x.disc, a.disc);
          x.count += a.count;
        }
      if (static_cast<int64_t>(all.size()) > out_rows) return -1;
      int64_t r = 0;
      for (const auto& [k, a] : all) {
        int64_t* o = out + r * 10;
        const double cnt = static_cast<double>(a.count);
        o[0] = k.first;
        o[1] = k.second;
        o[2] = a.qty;
        o[3] = a.price;
        o[4] = a.disc_price;
        o[5] = a.charge;
        o[6] = dbits(static_cast<double>(a.qty) / cnt);
        o[7] = dbits(static_cast<double>(a.price) / cnt);
        o[8] = dbits(static_cast<double>(a.disc) / cnt);
        o[9] = a.count;
        ++r;
      }
      return r;
    }
    case PORT_SSB11: {
      // ddate join (d_year = 1993), lo_discount between 1 and 3, lo_quantity < 25
      const int64_t nd = dim_rows[0];
      const int64_t* dkey = c[0];
      const int64_t* dyear = c[1];
      std::vector<bool> keep(static_cast<std::size_t>(nd));
      for (int64_t i = 0; i < nd; ++i) keep[static_cast<std::size_t>(i)] = dyear[i] == 1993;
      const std::vector<int32_t> idx = index_keys(dkey, nd, &keep);
      std::vector<int64_t> part(static_cast<std::size_t>(T), 0);
      feed(T, [&](int t, const int64_t* const* f, int64_t n) {
        int64_t s = 0;
        for (int64_t i = 0; i < n; ++i)
          if (f[1][i] >= 1 && f[1][i] <= 3 && f[2][i] < 25 && lookup(idx, f[0][i]) >= 0)
            s = wadd(s, wmul(f[3][i], f[1][i]));
        part[static_cast<std::size_t>(t)] = wadd(part[static_cast<std::size_t>(t)], s);
      });
      int64_t s = 0;
      for (int64_t p : part) s = wadd(s, p);
      if (out_rows < 1) return -1;
      out[0] = s;
      return 1;
    }
    case PORT_SSB41: {
      const int64_t nc = dim_rows[0], ns = dim_rows[1], np = dim_rows[2], nd = dim_rows[3];
      const int64_t *ckey = c[0], *creg = c[1], *cnat = c[2], *skey = c[3], *sreg = c[4],
                    *pkey = c[5], *pmfgr = c[6], *dkey = c[7], *dyear = c[8];
      std::vector<bool> kc(static_cast<std::size_t>(nc)), ks(static_cast<std::size_t>(ns)),
          kp(static_cast<std::size_t>(np));
      for (int64_t i = 0; i < nc; ++i) kc[static_cast<std::size_t>(i)] = creg[i] == codes[0];
      for (int64_t i = 0; i < ns; ++i) ks[static_cast<std::size_t>(i)] = sreg[i] == codes[1];
      for (int64_t i = 0; i < np; ++i)
        kp[static_cast<std::size_t>(i)] = pmfgr[i] != codes[2] && pmfgr[i] != codes[3] && pmfgr[i] != codes[4];
      const auto ic = index_keys(ckey, nc, &kc), is = index_keys(skey, ns, &ks),
                 ip = index_keys(pkey, np, &kp), id = index_keys(dkey, nd, nullptr);
      using Map = std::map<std::pair<int64_t, int64_t>, int64_t>;
      std::vector<Map> maps(static_cast<std::size_t>(T));
      feed(T, [&](int t, const int64_t* const* f, int64_t n) {
        Map& m = maps[static_cast<std::size_t>(t)];
        for (int64_t i = 0; i < n; ++i) {
          const int32_t rc = lookup(ic, f[0][i]);
          if (rc < 0) continue;
          if (lookup(is, f[1][i]) < 0) continue;
          if (lookup(ip, f[2][i]) < 0) continue;
          const int32_t rd = lookup(id, f[3][i]);
          if (rd < 0) continue;
          int64_t& v = m[{dyear[rd], cnat[rc]}];
          v = wadd(v, wsub(f[4][i], f[5][i]));
        }
      });
      Map all;
      for (const Map& m : maps)
        for (const auto& [k, v] : m) all[k] = wadd(all[k], v);
      if (static_cast<int64_t>(all.size()) > out_rows) return -1;
      int64_t r = 0;
      for (const auto& [k, v] : all) {
        out[r * 3 + 0] = k.first;
        out[r * 3 + 1] = k.second;
        out[r * 3 + 2] = v;
        ++r;
      }
      return r;
    }
    case PORT_Q3: {
      const int64_t no = dim_rows[0], nc = dim_rows[1];
      const int64_t *okey = c[0], *ocust = c[1], *odate = c[2], *oprio = c[3], *ckey = c[4],
                    *cseg = c[5];
      std::vector<bool> ko(static_cast<std::size_t>(no)), kc(static_cast<std::size_t>(nc));
      for (int64_t i = 0; i < no; ++i) ko[static_cast<std::size_t>(i)] = odate[i] < 19950315;
      for (int64_t i = 0; i < nc; ++i) kc[static_cast<std::size_t>(i)] = cseg[i] == codes[0];
      const auto io = index_keys(okey, no, &ko), ic = index_keys(ckey, nc, &kc);
      struct G { int64_t date, prio, rev; };
      using Map = std::unordered_map<int64_t, G>;
      std::vector<Map> maps(static_cast<std::size_t>(T));
      feed(T, [&](int t, const int64_t* const* f, int64_t n) {
        Map& m = maps[static_cast<std::size_t>(t)];
        for (int64_t i = 0; i < n; ++i) {
          if (!(f[1][i] > 19950315)) continue;
          const int32_t ro = lookup(io, f[0][i]);
          if (ro < 0) continue;
          if (lookup(ic, ocust[ro]) < 0) continue;
          auto [it, fresh] = m.try_emplace(f[0][i], G{odate[ro], oprio[ro], 0});
          it->second.rev = wadd(it->second.rev, wmul(f[2][i], wsub(100, f[3][i])));
        }
      });
      Map all;
      for (Map& m : maps) {
        for (const auto& [k, g] : m) {
          auto [it, fresh] = all.try_emplace(k, G{g.date, g.prio, 0});
          it->second.rev = wadd(it->second.rev, g.rev);
        }
        Map().swap(m);
      }
      if (static_cast<int64_t>(all.size()) > out_rows) return -1;
      int64_t r = 0;
      for (const auto& [k, g] : all) {
        out[r * 4 + 0] = k;
        out[r * 4 + 1] = g.rev;
        out[r * 4 + 2] = g.date;
        out[r * 4 + 3] = g.prio;
        ++r;
      }
      return r;
    }
  }
  return 0;
}

}  // namespace

extern "C" {

void port_gen(int table, int col, double sf, uint64_t seed, int64_t begin, int64_t n, int64_t* out,
              int threads) {
  parallel_for(n, threads, [&](int, int64_t b, int64_t e) {
    for (int64_t i = b; i < e; ++i) out[i] = hg_value(table, col, begin + i, sf, seed);
  });
}

int port_width(int query) {
  switch (query) {
    case PORT_Q6: return 1;
    case PORT_Q1: return 10;
    case PORT_SSB11: return 1;
    case PORT_SSB41: return 3;
    case PORT_Q3: return 4;
  }
  return 0;
}

int64_t port_run(int query, const int64_t* const* c, int64_t n, const int64_t* dim_rows,
                 const int64_t* codes, int threads, int64_t* out, int64_t out_rows) {
  if (query < PORT_Q6 || query > PORT_Q3) return -1;
  const std::size_t nf = fact_columns(query).size();
  const Feed feed = [&](int T, const Body& body) {
    parallel_for(n, T, [&](int t, int64_t b, int64_t e) {
      std::array<const int64_t*, 8> f{};
      for (std::size_t k = 0; k < nf; ++k) f[k] = c[k] + b;
      body(t, f.data(), e - b);
    });
  };
  return execute(query, c + nf, dim_rows, codes, std::max(1, threads), feed, out, out_rows);
}

int64_t port_run_gen(int query, double sf, uint64_t seed, int64_t row_begin, int64_t n,
                     const int64_t* codes, int threads, int64_t* out, int64_t out_rows) {
  if (query < PORT_Q6 || query > PORT_Q3) return -1;
  const int T = std::max(1, threads);
  // dimension tables, whole
  const auto& dcols = dim_columns(query);
  std::vector<std::vector<int64_t>> dims(dcols.size());
  std::vector<const int64_t*> dptr(dcols.size());
  for (std::size_t k = 0; k < dcols.size(); ++k) {
    const int64_t rows = hg_table_rows(dcols[k].table, sf);
    dims[k].resize(static_cast<std::size_t>(rows));
    port_gen(dcols[k].table, dcols[k].col, sf, seed, 0, rows, dims[k].data(), T);
    dptr[k] = dims[k].data();
  }
  std::vector<int64_t> dim_rows;
  for (int t : dim_tables(query)) dim_rows.push_back(hg_table_rows(t, sf));
  // fact rows, regenerated per chunk by each worker
  const auto& fcols = fact_columns(query);
  const Feed feed = [&](int Tn, const Body& body) {
    parallel_for(n, Tn, [&](int t, int64_t b, int64_t e) {
      constexpr int64_t kChunk = 1 << 14;
      std::vector<std::vector<int64_t>> buf(fcols.size(), std::vector<int64_t>(kChunk));
      std::array<const int64_t*, 8> f{};
      for (int64_t cb = b; cb < e; cb += kChunk) {
        const int64_t len = std::min(kChunk, e - cb);
        for (std::size_t k = 0; k < fcols.size(); ++k) {
          int64_t* o = buf[k].data();
          for (int64_t i = 0; i < len; ++i) o[i] = hg_value(fcols[k].table, fcols[k].col, row_begin + cb + i, sf, seed);
          f[k] = o;
        }
        body(t, f.data(), len);
      }
    });
  };
  return execute(query, dptr.data(), dim_rows.data(), codes, T, feed, out, out_rows);
}

}  // extern "C"
