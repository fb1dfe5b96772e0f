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

// dataset.cpp:193-205: comma split, each field trimmed of " \t\r", a trailing comma adds an empty field
std::vector<std::string> split_csv_line(const std::string& line) {
  std::vector<std::string> out;
  std::string field;
  std::stringstream ss(line);
  while (std::getline(ss, field, ',')) {
    const auto b = field.find_first_not_of(" \t\r");
    const auto e = field.find_last_not_of(" \t\r");
    out.push_back(b == std::string::npos ? std::string() : field.substr(b, e - b + 1));
  }
  if (!line.empty() && line.back() == ',') out.emplace_back();
  return out;
}

// dataset.cpp:207-218: the whole field must parse (std::stod) to a finite value
double parse_num(const std::string& s, const std::string& path, int lineno) {
  try {
    std::size_t pos = 0;
    const double v = std::stod(s, &pos);
    if (pos != s.size()) throw std::invalid_argument(s);
    if (!std::isfinite(v)) throw std::invalid_argument(s);
    return v;
  } catch (const std::exception&) {
    data_error(path + ":" + std::to_string(lineno) + ": missing or non-numeric value '" + s + "'");
  }
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

// read_dataset_csv (dataset.cpp:221-296)
int stgp_read_dataset_csv(const char* path_c, stgp_table** out) {
  using namespace stgp;
  return guarded([&] {
    if (!path_c || !out) config_error("stgp_read_dataset_csv: null argument");
    const std::string path(path_c);
    std::ifstream is(path);
    if (!is) data_error("cannot open dataset: " + path);
    std::string line;
    int lineno = 0;
    std::vector<std::string> header;
    while (std::getline(is, line)) {
      ++lineno;
      if (line.empty() || line[0] == '#') continue;
      header = split_csv_line(line);
      break;
    }
    if (header.empty()) data_error(path + ": missing header row");
    int cx = -1, cy = -1, ct = -1, cv = -1, cs = -1;
    std::vector<int> cov;
    auto tab = std::make_unique<stgp_table>();
    for (int j = 0; j < static_cast<int>(header.size()); ++j) {
      const std::string& name = header[static_cast<size_t>(j)];
      if (name == "x") cx = j;
      else if (name == "y") cy = j;
      else if (name == "t") ct = j;
      else if (name == "value") cv = j;
      else if (name == "station_id") cs = j;
      else {
        cov.push_back(j);
        tab->covariate_names.push_back(name);
      }
    }
    if (cx < 0 || cy < 0 || ct < 0 || cv < 0) data_error(path + ": required columns are x, y, t, value");
    std::vector<double> covr;  // row-major
    while (std::getline(is, line)) {
      ++lineno;
      if (line.empty() || line[0] == '#') continue;
      const auto f = split_csv_line(line);
      if (f.size() != header.size())
        data_error(path + ":" + std::to_string(lineno) + ": expected " + std::to_string(header.size()) + " fields");
      const double x = parse_num(f[static_cast<size_t>(cx)], path, lineno);
      const double y = parse_num(f[static_cast<size_t>(cy)], path, lineno);
      const double t = parse_num(f[static_cast<size_t>(ct)], path, lineno);
      const double v = parse_num(f[static_cast<size_t>(cv)], path, lineno);
      tab->x.push_back(x);
      tab->y.push_back(y);
      tab->t.push_back(t);
      tab->value.push_back(v);
      if (cs >= 0) {
        const std::string& s = f[static_cast<size_t>(cs)];
        if (s.empty()) data_error(path + ":" + std::to_string(lineno) + ": empty station_id");
        tab->stations.push_back(s);
      }
      for (int j : cov) covr.push_back(parse_num(f[static_cast<size_t>(j)], path, lineno));
    }
    if (tab->x.empty()) data_error(path + ": no data rows");
    tab->n = static_cast<int>(tab->x.size());
    tab->p = static_cast<int>(cov.size());
    tab->X.assign(static_cast<size_t>(tab->n) * tab->p, 0.0);
    for (int i = 0; i < tab->n; ++i)
      for (int j = 0; j < tab->p; ++j)
        tab->X[static_cast<size_t>(j) * tab->n + i] = covr[static_cast<size_t>(i) * tab->p + j];
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
