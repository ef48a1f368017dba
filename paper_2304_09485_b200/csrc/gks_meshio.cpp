// Native ugks-mesh reader (replaces the per-line Python parse of
// gks3d/mesh/fileio.py:42-103 for 10^7-cell meshes).
//
// Grammar (fileio.py): comment = '#' to end of line; blank lines skipped;
//   ugks-mesh 1
//   nodes N      + N lines "x y z"
//   tets T       + T lines of 4 node ids
//   hexes H      + H lines of 8 node ids
//   patches P    + per patch "<name> <faces>" + that many lines of 3 or 4 ids
// On any grammar violation the reader returns GKS_ERR_BAD_ARG; the Python
// caller then re-parses with the reference-shaped parser to raise the
// reference's exact MeshError (mesh.py load_mesh), so only the fast path
// lives here.
#include <errno.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <string>
#include <vector>

#include "../../include/gks.h"

struct GksUgks {
  std::vector<double> nodes;
  std::vector<int64_t> tets, hexes;
  std::vector<std::string> names;
  std::vector<int64_t> counts;     // faces per patch
  std::vector<int64_t> faces;      // (sum counts, 4), -1 padded
  std::vector<int8_t> widths;      // 3 or 4 per face
};

namespace {

struct Lines {
  const char* p;
  const char* end;
  // next non-empty logical line (comment stripped); false at end of input
  bool next(const char** b, const char** e) {
    while (p < end) {
      const char* ls = p;
      const char* le = (const char*)memchr(p, '\n', (size_t)(end - p));
      if (!le) le = end;
      p = le < end ? le + 1 : end;
      const char* h = (const char*)memchr(ls, '#', (size_t)(le - ls));
      if (h) le = h;
      while (ls < le && (*ls == ' ' || *ls == '\t' || *ls == '\r' || *ls == '\f' || *ls == '\v')) ++ls;
      while (le > ls && (le[-1] == ' ' || le[-1] == '\t' || le[-1] == '\r' || le[-1] == '\f' || le[-1] == '\v')) --le;
      if (ls < le) {
        *b = ls;
        *e = le;
        return true;
      }
    }
    return false;
  }
};

inline bool ws(char c) { return c == ' ' || c == '\t' || c == '\r' || c == '\f' || c == '\v'; }

// split [b, e) into at most `cap` tokens; returns the token count (cap + 1 if more)
int split(const char* b, const char* e, const char** tb, const char** te, int cap) {
  int n = 0;
  while (b < e) {
    while (b < e && ws(*b)) ++b;
    if (b >= e) break;
    const char* s = b;
    while (b < e && !ws(*b)) ++b;
    if (n == cap) return cap + 1;
    tb[n] = s;
    te[n] = b;
    ++n;
  }
  return n;
}

bool to_f64(const char* b, const char* e, double* out) {
  char buf[64];
  const size_t n = (size_t)(e - b);
  if (n == 0 || n >= sizeof(buf)) return false;
  memcpy(buf, b, n);
  buf[n] = 0;
  char* end = nullptr;
  errno = 0;
  *out = strtod(buf, &end);
  return end == buf + n;
}

bool to_i64(const char* b, const char* e, int64_t* out) {
  char buf[32];
  const size_t n = (size_t)(e - b);
  if (n == 0 || n >= sizeof(buf)) return false;
  memcpy(buf, b, n);
  buf[n] = 0;
  char* end = nullptr;
  errno = 0;
  *out = strtoll(buf, &end, 10);
  return end == buf + n && errno == 0;
}

bool counted(Lines& L, const char* tag, int64_t* n) {
  const char *b, *e, *tb[3], *te[3];
  if (!L.next(&b, &e)) return false;
  if (split(b, e, tb, te, 2) != 2) return false;
  if ((size_t)(te[0] - tb[0]) != strlen(tag) || memcmp(tb[0], tag, strlen(tag)) != 0) return false;
  return to_i64(tb[1], te[1], n) && *n >= 0;
}

template <class T, class Conv>
bool block(Lines& L, int64_t count, int width, std::vector<T>& out, Conv conv) {
  out.resize((size_t)count * width);
  const char *b, *e, *tb[9], *te[9];
  for (int64_t i = 0; i < count; ++i) {
    if (!L.next(&b, &e)) return false;
    if (split(b, e, tb, te, width) != width) return false;
    for (int k = 0; k < width; ++k)
      if (!conv(tb[k], te[k], &out[(size_t)i * width + k])) return false;
  }
  return true;
}

}  // namespace

extern "C" {

int gks_ugks_read(const char* path, GksUgks** out) {
  if (!path || !out) return GKS_ERR_BAD_ARG;
  FILE* fh = fopen(path, "rb");
  if (!fh) return GKS_ERR_BAD_ARG;
  std::string buf;
  fseek(fh, 0, SEEK_END);
  const long sz = ftell(fh);
  fseek(fh, 0, SEEK_SET);
  buf.resize(sz > 0 ? (size_t)sz : 0);
  const size_t got = sz > 0 ? fread(&buf[0], 1, (size_t)sz, fh) : 0;
  fclose(fh);
  if ((long)got != sz) return GKS_ERR_BAD_ARG;
  Lines L{buf.data(), buf.data() + buf.size()};
  GksUgks* m = new GksUgks();
  auto fail = [&]() {
    delete m;
    return GKS_ERR_BAD_ARG;
  };
  {
    const char *b, *e, *tb[3], *te[3];
    if (!L.next(&b, &e) || split(b, e, tb, te, 2) != 2) return fail();
    if (std::string(tb[0], te[0]) != "ugks-mesh" || std::string(tb[1], te[1]) != "1") return fail();
  }
  int64_t n;
  if (!counted(L, "nodes", &n) || !block(L, n, 3, m->nodes, to_f64)) return fail();
  if (!counted(L, "tets", &n) || !block(L, n, 4, m->tets, to_i64)) return fail();
  if (!counted(L, "hexes", &n) || !block(L, n, 8, m->hexes, to_i64)) return fail();
  int64_t np_;
  if (!counted(L, "patches", &np_)) return fail();
  for (int64_t p = 0; p < np_; ++p) {
    const char *b, *e, *tb[5], *te[5];
    if (!L.next(&b, &e) || split(b, e, tb, te, 2) != 2) return fail();
    std::string name(tb[0], te[0]);
    int64_t nf;
    if (!to_i64(tb[1], te[1], &nf)) return fail();
    for (const std::string& s : m->names)
      if (s == name) return fail();  // duplicate patch name
    m->names.push_back(name);
    m->counts.push_back(nf < 0 ? 0 : nf);
    for (int64_t f = 0; f < nf; ++f) {
      if (!L.next(&b, &e)) return fail();
      const int k = split(b, e, tb, te, 4);
      if (k != 3 && k != 4) return fail();
      int64_t ids[4] = {-1, -1, -1, -1};
      for (int t = 0; t < k; ++t)
        if (!to_i64(tb[t], te[t], &ids[t])) return fail();
      m->faces.insert(m->faces.end(), ids, ids + 4);
      m->widths.push_back((int8_t)k);
    }
  }
  *out = m;
  return GKS_OK;
}

int gks_ugks_sizes(const GksUgks* m, int64_t* nnodes, int64_t* ntets, int64_t* nhexes, int64_t* npatches) {
  if (!m) return GKS_ERR_BAD_ARG;
  if (nnodes) *nnodes = (int64_t)m->nodes.size() / 3;
  if (ntets) *ntets = (int64_t)m->tets.size() / 4;
  if (nhexes) *nhexes = (int64_t)m->hexes.size() / 8;
  if (npatches) *npatches = (int64_t)m->names.size();
  return GKS_OK;
}

int gks_ugks_patch(const GksUgks* m, int64_t k, char* name, int64_t cap, int64_t* nfaces) {
  if (!m || k < 0 || k >= (int64_t)m->names.size()) return GKS_ERR_BAD_ARG;
  if (name && cap > 0) {
    snprintf(name, (size_t)cap, "%s", m->names[k].c_str());
  }
  if (nfaces) *nfaces = m->counts[k];
  return GKS_OK;
}

int gks_ugks_copy(const GksUgks* m, double* nodes, int64_t* tets, int64_t* hexes, int64_t* faces, int8_t* widths) {
  if (!m) return GKS_ERR_BAD_ARG;
  if (nodes && !m->nodes.empty()) memcpy(nodes, m->nodes.data(), m->nodes.size() * sizeof(double));
  if (tets && !m->tets.empty()) memcpy(tets, m->tets.data(), m->tets.size() * sizeof(int64_t));
  if (hexes && !m->hexes.empty()) memcpy(hexes, m->hexes.data(), m->hexes.size() * sizeof(int64_t));
  if (faces && !m->faces.empty()) memcpy(faces, m->faces.data(), m->faces.size() * sizeof(int64_t));
  if (widths && !m->widths.empty()) memcpy(widths, m->widths.data(), m->widths.size());
  return GKS_OK;
}

void gks_ugks_free(GksUgks* m) { delete m; }

}  // extern "C"
