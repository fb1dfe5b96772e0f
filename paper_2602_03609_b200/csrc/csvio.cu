// Dataset CSV and neighbour-audit formats, byte-compatible with the
// reference: read_dataset_csv / write_dataset_csv (dataset.cpp:191-316) and
// write_neighbor_debug_csv (neighbors.cpp:336-355, the metrics of cli.cpp:516-572).
// Host code: parsing and formatting only; the neighbour distances come from the device searches.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <sstream>
#include <string>
#include <vector>

#include "structure.hpp"
#include "../../include/stgp_b200.h"

struct stgp_table {
  int n = 0, p = 0;
  std::vector<double> x, y, t, value, X;  // X: n x p column-major
  std::vector<std::string> stations, covariate_names;
};

namespace stgp {
namespace {

template <class F>
int guarded(F&& f) {
  try {
    f();
    return STGP_OK;
  } catch (const Error& e) {
    g_last_error = e.what();
    return e.code;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return STGP_ERR_INTERNAL;
  }
}

// Format contract (exercised by test_dataset.cpp:146-189): '#'-prefixed and empty lines are
// skipped; the first other line is the header; cells are comma separated and stripped of blanks
// (space, tab, CR) at both ends; a row must have as many cells as the header.  The whole file is read
// into one buffer and scanned in place: a cursor walks the lines, and each line is cut into cell views.
struct Cell {
  const char* p;
  size_t len;
  std::string str() const { return std::string(p, len); }
  bool is(const char* name) const { return std::strlen(name) == len && std::memcmp(p, name, len) == 0; }
};

inline bool blank(char c) { return c == ' ' || c == '\t' || c == '\r'; }

// cells of [b, e): every comma ends one cell, so "a,b," has three (the last empty)
void cut_cells(const char* b, const char* e, std::vector<Cell>& cells) {
  cells.clear();
  const char* c = b;
  for (;;) {
    const char* stop = static_cast<const char*>(std::memchr(c, ',', static_cast<size_t>(e - c)));
    const char* ce = stop ? stop : e;
    const char* lo = c;
    const char* hi = ce;
    while (lo < hi && blank(*lo)) ++lo;
    while (hi > lo && blank(hi[-1])) --hi;
    cells.push_back(Cell{lo, static_cast<size_t>(hi - lo)});
    if (!stop) break;
    c = stop + 1;
  }
}

struct LineCursor {
  const std::string& buf;
  size_t pos = 0;
  int lineno = 0;
  // next line that is neither empty nor a '#' comment; false at end of input
  bool next(const char*& b, const char*& e) {
    while (pos < buf.size()) {
      const size_t nl = buf.find('\n', pos);
      const size_t stop = nl == std::string::npos ? buf.size() : nl;
      b = buf.data() + pos;
      e = buf.data() + stop;
      pos = stop + 1;
      ++lineno;
      if (e > b && *b != '#') return true;
    }
    return false;
  }
};

// a cell that holds exactly one finite number (strtod must consume all of it)
double number_cell(const Cell& c, const std::string& where) {
  char tmp[128];
  bool ok = c.len > 0 && c.len < sizeof(tmp);
  double v = 0.0;
  if (ok) {
    std::memcpy(tmp, c.p, c.len);
    tmp[c.len] = '\0';
    char* end = nullptr;
    v = std::strtod(tmp, &end);
    ok = end == tmp + c.len && std::isfinite(v) && !blank(tmp[0]);
  }
  if (!ok) data_error(where + ": value '" + c.str() + "' is empty or not a finite number");
  return v;
}

// std::ostream with precision(17) and the default float field: "%.17g"
void put_num(std::string& o, double v) {
  char buf[64];
  std::snprintf(buf, sizeof(buf), "%.17g", v);
  o += buf;
}

int copy_str(const std::string& s, char* buf, int cap) {
  if (buf && cap > 0) {
    const int k = std::min(cap - 1, static_cast<int>(s.size()));
    std::memcpy(buf, s.data(), static_cast<size_t>(k));
    buf[k] = '\0';
  }
  return static_cast<int>(s.size());
}

}  // namespace
}  // namespace stgp

extern "C" {

// read_dataset_csv (dataset.cpp:221-296): columns x, y, t, value required, station_id optional, every
// other column a numeric covariate in header order.
int stgp_read_dataset_csv(const char* path_c, stgp_table** out) {
  using namespace stgp;
  return guarded([&] {
    if (!path_c || !out) config_error("stgp_read_dataset_csv: null argument");
    const std::string path(path_c);
    std::string buf;
    {
      std::ifstream is(path, std::ios::binary);
      if (!is) data_error("dataset " + path + " cannot be opened");
      std::ostringstream ss;
      ss << is.rdbuf();
      buf = ss.str();
    }
    LineCursor cur{buf};
    const char *b = nullptr, *e = nullptr;
    if (!cur.next(b, e)) data_error(path + ": no header line");
    std::vector<Cell> cells;
    cut_cells(b, e, cells);
    const size_t width = cells.size();
    enum Role { kX, kY, kT, kValue, kStation, kCovariate };
    std::vector<int> role(width);
    int have[5] = {0, 0, 0, 0, 0};
    auto tab = std::make_unique<stgp_table>();
    static const char* const kNames[5] = {"x", "y", "t", "value", "station_id"};
    for (size_t j = 0; j < width; ++j) {
      int r = kCovariate;
      for (int q = 0; q < 5; ++q)
        if (cells[j].is(kNames[q])) r = q;
      role[j] = r;
      if (r == kCovariate) tab->covariate_names.push_back(cells[j].str());
      else ++have[r];
    }
    if (!have[kX] || !have[kY] || !have[kT] || !have[kValue])
      data_error(path + ": header lacks one of the required columns x, y, t, value");
    const int p = static_cast<int>(tab->covariate_names.size());
    std::vector<double> cov_rows;  // row-major while reading
    while (cur.next(b, e)) {
      cut_cells(b, e, cells);
      const std::string where = path + ":" + std::to_string(cur.lineno);
      if (cells.size() != width)
        data_error(where + ": " + std::to_string(cells.size()) + " cells, the header has " + std::to_string(width));
      double v[4] = {0, 0, 0, 0};
      std::string station;
      for (size_t j = 0; j < width; ++j) {  // a repeated header name: the last column of that name wins
        switch (role[j]) {
          case kStation:
            if (cells[j].len == 0) data_error(where + ": station_id is empty");
            station = cells[j].str();
            break;
          case kCovariate: cov_rows.push_back(number_cell(cells[j], where)); break;
          default: v[role[j]] = number_cell(cells[j], where);
        }
      }
      tab->x.push_back(v[kX]);
      tab->y.push_back(v[kY]);
      tab->t.push_back(v[kT]);
      tab->value.push_back(v[kValue]);
      if (have[kStation]) tab->stations.push_back(std::move(station));
    }
    if (tab->x.empty()) data_error(path + ": header but no observations");
    tab->n = static_cast<int>(tab->x.size());
    tab->p = p;
    tab->X.resize(static_cast<size_t>(tab->n) * p);
    for (int i = 0; i < tab->n; ++i)
      for (int j = 0; j < p; ++j) tab->X[static_cast<size_t>(j) * tab->n + i] = cov_rows[static_cast<size_t>(i) * p + j];
    *out = tab.release();
  });
}

int stgp_table_shape(const stgp_table* tab, int* n, int* p, int* has_stations) {
  if (!tab) return STGP_ERR_CONFIG;
  if (n) *n = tab->n;
  if (p) *p = tab->p;
  if (has_stations) *has_stations = tab->stations.empty() ? 0 : 1;
  return STGP_OK;
}

int stgp_table_columns(const stgp_table* tab, double* x, double* y, double* t, double* value, double* X) {
  if (!tab) return STGP_ERR_CONFIG;
  if (x) std::copy(tab->x.begin(), tab->x.end(), x);
  if (y) std::copy(tab->y.begin(), tab->y.end(), y);
  if (t) std::copy(tab->t.begin(), tab->t.end(), t);
  if (value) std::copy(tab->value.begin(), tab->value.end(), value);
  if (X) std::copy(tab->X.begin(), tab->X.end(), X);
  return STGP_OK;
}

int stgp_table_station(const stgp_table* tab, int i, char* buf, int cap) {
  if (!tab || i < 0 || i >= static_cast<int>(tab->stations.size())) return -1;
  return stgp::copy_str(tab->stations[static_cast<size_t>(i)], buf, cap);
}

int stgp_table_covariate_name(const stgp_table* tab, int j, char* buf, int cap) {
  if (!tab || j < 0 || j >= tab->p) return -1;
  return stgp::copy_str(tab->covariate_names[static_cast<size_t>(j)], buf, cap);
}

void stgp_table_destroy(stgp_table* tab) { delete tab; }

// write_dataset_csv (dataset.cpp:298-316)
int stgp_write_dataset_csv(const char* path_c, int n, const double* x, const double* y, const double* t,
                           const double* value, int p, const double* X, const char* const* stations,
                           const char* header_comment) {
  using namespace stgp;
  return guarded([&] {
    if (!path_c || n < 0 || (n > 0 && (!x || !y || !t || !value)) || (p > 0 && !X)) config_error("stgp_write_dataset_csv: bad argument");
    std::ofstream os(path_c, std::ios::binary);
    if (!os) data_error(std::string("cannot open output dataset: ") + path_c);
    std::string o;
    if (header_comment && *header_comment) o += std::string("# ") + header_comment + "\n";
    o += "x,y,t,value";
    if (stations) o += ",station_id";
    for (int j = 0; j < p; ++j) o += ",x" + std::to_string(j);
    o += "\n";
    for (int i = 0; i < n; ++i) {
      put_num(o, x[i]);
      o += ',';
      put_num(o, y[i]);
      o += ',';
      put_num(o, t[i]);
      o += ',';
      put_num(o, value[i]);
      if (stations) {
        o += ',';
        o += stations[i];
      }
      for (int j = 0; j < p; ++j) {
        o += ',';
        put_num(o, X[static_cast<size_t>(j) * n + i]);
      }
      o += '\n';
    }
    os << o;
  });
}

// write_neighbor_debug_csv (neighbors.cpp:336-355): per row i its set sorted by (metric(i, j), j).
// d_c / d_r: the searches' distances (bit-identical to DcMetric / DrMetric); euclid: the scaled
// metric of cli.cpp:549-563 recomputed on the host from the ordered coordinates.
int stgp_write_neighbor_debug_csv(const char* path_c, const stgp_neighbors* nb, const stgp_dataset* ds,
                                  const char* header_comment) {
  using namespace stgp;
  return guarded([&] {
    if (!path_c || !nb || !ds || ds->n != nb->n) config_error("stgp_write_neighbor_debug_csv: bad argument");
    const int n = nb->n, m = nb->m_v;
    std::vector<int32_t> idx(static_cast<size_t>(n) * m);
    std::vector<double> dist(static_cast<size_t>(n) * m);
    nb->idx.download(idx.data(), idx.size(), nb->ctx->stream);
    const bool euclid = nb->kind == STGP_METRIC_EUCLID;
    if (!euclid) {
      if (!nb->has_dist) config_error("these neighbour sets carry no distances");
      nb->dist.download(dist.data(), dist.size(), nb->ctx->stream);
    }
    STGP_CUDA(cudaStreamSynchronize(nb->ctx->stream));
    std::ofstream os(path_c, std::ios::binary);
    if (!os) config_error(std::string("cannot open neighbor audit file: ") + path_c);
    std::string o;
    if (header_comment && *header_comment) o += std::string("# ") + header_comment + "\n";
    o += "i,rank,neighbor_index,distance\n";
    std::vector<std::pair<double, int>> by;
    for (int i = 0; i < n; ++i) {
      by.clear();
      for (int a = 0; a < m; ++a) {
        const int j = idx[static_cast<size_t>(i) * m + a];
        if (j < 0) continue;
        double d;
        if (euclid) {
          const double dx = (ds->hx[i] - ds->hx[j]) / nb->ss, dy = (ds->hy[i] - ds->hy[j]) / nb->ss,
                       dt = (ds->ht[i] - ds->ht[j]) / nb->ts;
          d = std::sqrt(dx * dx + dy * dy + dt * dt);
        } else {
          d = dist[static_cast<size_t>(i) * m + a];
        }
        by.emplace_back(d, j);
      }
      std::sort(by.begin(), by.end());
      for (size_t r = 0; r < by.size(); ++r) {
        o += std::to_string(i) + "," + std::to_string(r) + "," + std::to_string(by[r].second) + ",";
        put_num(o, by[r].first);
        o += '\n';
      }
    }
    os << o;
  });
}

}  // extern "C"
