/* pyhost.c -- CPython helpers of the host path (module _pyhost).
 *
 * Two places where the public Python API (align.mine_corpus, SURVEY.md
 * section 8 f2/f3) would otherwise loop over ~10^6 Python objects:
 *
 *   str_view(sentences, ptrs, lens, prefix) -> bool
 *       The characters of every sentence in place, for the native tokenizer
 *       (bimine_tokenize_ptrs): ptrs[k] / lens[k] the storage and length of
 *       sentences[k], prefix[k] = sum(lens[:k]).  False (buffers partly
 *       written) unless every item is an exact, compact ASCII str -- the
 *       caller then encodes the sentences to one UTF-8 buffer instead.  The
 *       caller keeps the list alive while the pointers are used.
 *
 *   docs_view(docs, ptrs, lens, prefix, start) -> bool
 *       The same over a list of document pairs (source sentences, target
 *       sentences), each a tuple or list, each side a tuple or list of str:
 *       pair by pair, source then target sentences -- no flat list of
 *       10^6 sentences to build and free; pair d's first sentence is
 *       start[d] (start[n_docs] = the total).  Ranges of pairs on up to 16
 *       threads.  False also for any other shape or counts.
 *
 *   build_rows(matches, counts, pair, docs) -> list
 *       The mining rows (score, source sentence, target sentence) of
 *       align.py:441-447, in pair order: the k-th mined pair, docs[pair[k]],
 *       owns the next counts[k] records of `matches` (bimine_match: f64
 *       score, i32 i, i32 j): source sentence i, target sentence j.
 */
#define PY_SSIZE_T_CLEAN
#include <Python.h>
#include <pthread.h>
#include <stdint.h>
#include <string.h>

/* items of an exact tuple or list (borrowed), else NULL */
static PyObject **seq_items(PyObject *o, Py_ssize_t *n) {
  if (PyTuple_CheckExact(o)) {
    *n = PyTuple_GET_SIZE(o);
    return &PyTuple_GET_ITEM(o, 0);
  }
  if (PyList_CheckExact(o)) {
    *n = PyList_GET_SIZE(o);
    return ((PyListObject *)o)->ob_item;
  }
  return NULL;
}

static int get_buf(PyObject *o, Py_buffer *b, int writable, Py_ssize_t itemsize, const char *name) {
  if (PyObject_GetBuffer(o, b, (writable ? PyBUF_WRITABLE : 0) | PyBUF_C_CONTIGUOUS) < 0) return -1;
  if (itemsize && b->len % itemsize) {
    PyErr_Format(PyExc_ValueError, "%s: buffer of %zd bytes is not a whole number of %zd-byte items", name, b->len,
                 itemsize);
    PyBuffer_Release(b);
    return -1;
  }
  return 0;
}

static PyObject *str_view(PyObject *self, PyObject *args) {
  PyObject *list, *po, *lo, *xo;
  if (!PyArg_ParseTuple(args, "O!OOO", &PyList_Type, &list, &po, &lo, &xo)) return NULL;
  Py_buffer bp, bl, bx;
  if (get_buf(po, &bp, 1, 8, "ptrs") < 0) return NULL;
  if (get_buf(lo, &bl, 1, 8, "lens") < 0) {
    PyBuffer_Release(&bp);
    return NULL;
  }
  if (get_buf(xo, &bx, 1, 8, "prefix") < 0) {
    PyBuffer_Release(&bp);
    PyBuffer_Release(&bl);
    return NULL;
  }
  const Py_ssize_t n = PyList_GET_SIZE(list);
  int ok = 1;
  if (bp.len < 8 * n || bl.len < 8 * n || bx.len < 8 * (n + 1)) {
    PyErr_SetString(PyExc_ValueError, "str_view: output buffers are too small");
    ok = -1;
  } else {
    int64_t *P = (int64_t *)bp.buf, *L = (int64_t *)bl.buf, *X = (int64_t *)bx.buf;
    X[0] = 0;
    for (Py_ssize_t k = 0; k < n; ++k) {
      PyObject *o = PyList_GET_ITEM(list, k);
      if (!PyUnicode_CheckExact(o) || !PyUnicode_IS_COMPACT_ASCII(o)) {
        ok = 0;
        break;
      }
      P[k] = (int64_t)(intptr_t)PyUnicode_DATA(o);
      L[k] = (int64_t)PyUnicode_GET_LENGTH(o);
      X[k + 1] = X[k] + L[k];
    }
  }
  PyBuffer_Release(&bp);
  PyBuffer_Release(&bl);
  PyBuffer_Release(&bx);
  if (ok < 0) return NULL;
  return PyBool_FromLong(ok);
}

/* docs_view's work on docs [d0, d1): sentence s of doc d is written at
   start[d] + s.  Reads object memory only (no Python API calls), so the
   ranges run on plain threads while the caller holds the list. */
struct DocsRange {
  PyObject **docs;
  const int64_t *start;
  Py_ssize_t d0, d1, cap;
  int64_t *P, *L;
  int ok;
};

static void *docs_range(void *arg) {
  struct DocsRange *r = (struct DocsRange *)arg;
  for (Py_ssize_t d = r->d0; r->ok && d < r->d1; ++d) {
    Py_ssize_t two, s = r->start[d];
    PyObject **side = seq_items(r->docs[d], &two);
    if (!side || two != 2) {
      r->ok = 0;
      break;
    }
    for (int h = 0; r->ok && h < 2; ++h) {
      Py_ssize_t m;
      PyObject **it = seq_items(side[h], &m);
      if (!it) {
        r->ok = 0;
        break;
      }
      for (Py_ssize_t k = 0; k < m; ++k, ++s) {
        PyObject *o = it[k];
        if (s >= r->start[d + 1] || s >= r->cap || !PyUnicode_CheckExact(o) || !PyUnicode_IS_COMPACT_ASCII(o)) {
          r->ok = 0;
          break;
        }
        r->P[s] = (int64_t)(intptr_t)PyUnicode_DATA(o);
        r->L[s] = (int64_t)PyUnicode_GET_LENGTH(o);
      }
    }
    if (r->ok && s != r->start[d + 1]) r->ok = 0;  /* the caller's counts disagree with the docs */
  }
  return NULL;
}

static PyObject *docs_view(PyObject *self, PyObject *args) {
  PyObject *docs, *po, *lo, *xo, *so;
  if (!PyArg_ParseTuple(args, "O!OOOO", &PyList_Type, &docs, &po, &lo, &xo, &so)) return NULL;
  Py_buffer bp, bl, bx, bs;
  if (get_buf(po, &bp, 1, 8, "ptrs") < 0) return NULL;
  if (get_buf(lo, &bl, 1, 8, "lens") < 0) {
    PyBuffer_Release(&bp);
    return NULL;
  }
  if (get_buf(xo, &bx, 1, 8, "prefix") < 0) {
    PyBuffer_Release(&bp);
    PyBuffer_Release(&bl);
    return NULL;
  }
  if (get_buf(so, &bs, 0, 8, "start") < 0) {
    PyBuffer_Release(&bp);
    PyBuffer_Release(&bl);
    PyBuffer_Release(&bx);
    return NULL;
  }
  const Py_ssize_t nd = PyList_GET_SIZE(docs);
  const int64_t *start = (const int64_t *)bs.buf;
  int64_t *P = (int64_t *)bp.buf, *L = (int64_t *)bl.buf, *X = (int64_t *)bx.buf;
  const Py_ssize_t cap = bp.len / 8 < bl.len / 8 ? bp.len / 8 : bl.len / 8;
  int ok = bs.len / 8 == nd + 1 && start[0] == 0 && bx.len / 8 >= start[nd] + 1 && start[nd] <= cap;
  if (ok && nd > 0) {
    /* up to 16 ranges of >= 256 documents each */
    int nt = (int)(nd / 256);
    if (nt < 1) nt = 1;
    if (nt > 16) nt = 16;
    struct DocsRange r[16];
    pthread_t th[16];
    int started[16] = {0};
    for (int t = 0; t < nt; ++t) {
      r[t].docs = ((PyListObject *)docs)->ob_item;
      r[t].start = start;
      r[t].d0 = nd * t / nt;
      r[t].d1 = nd * (t + 1) / nt;
      r[t].cap = cap;
      r[t].P = P;
      r[t].L = L;
      r[t].ok = 1;
    }
    for (int t = 1; t < nt; ++t) started[t] = pthread_create(&th[t], NULL, docs_range, &r[t]) == 0;
    docs_range(&r[0]);
    for (int t = 1; t < nt; ++t) {
      if (started[t]) pthread_join(th[t], NULL);
      else docs_range(&r[t]);
    }
    for (int t = 0; t < nt; ++t) ok = ok && r[t].ok;
  }
  if (ok) {
    X[0] = 0;
    for (int64_t s = 0; s < start[nd]; ++s) X[s + 1] = X[s] + L[s];
  }
  PyBuffer_Release(&bp);
  PyBuffer_Release(&bl);
  PyBuffer_Release(&bx);
  PyBuffer_Release(&bs);
  return PyBool_FromLong(ok);
}

static PyObject *build_rows(PyObject *self, PyObject *args) {
  PyObject *mo, *co, *qo, *docs;
  if (!PyArg_ParseTuple(args, "OOOO!", &mo, &co, &qo, &PyList_Type, &docs)) return NULL;
  Py_buffer bm, bc, bq;
  if (get_buf(mo, &bm, 0, 16, "matches") < 0) return NULL;
  if (get_buf(co, &bc, 0, 8, "counts") < 0) goto fail_m;
  if (get_buf(qo, &bq, 0, 8, "pair") < 0) goto fail_c;
  {
    const Py_ssize_t K = bc.len / 8, total = bm.len / 16, nd = PyList_GET_SIZE(docs);
    const int64_t *cnt = (const int64_t *)bc.buf, *pq = (const int64_t *)bq.buf;
    const char *m = (const char *)bm.buf;
    if (bq.len / 8 != K) {
      PyErr_SetString(PyExc_ValueError, "build_rows: counts and pair differ in length");
      goto fail_all;
    }
    int64_t sum = 0;
    for (Py_ssize_t k = 0; k < K; ++k) {
      if (cnt[k] < 0) {
        PyErr_SetString(PyExc_ValueError, "build_rows: negative count");
        goto fail_all;
      }
      sum += cnt[k];
    }
    if (sum != total) {
      PyErr_Format(PyExc_ValueError, "build_rows: counts sum to %lld, %zd matches", (long long)sum, total);
      goto fail_all;
    }
    PyObject *out = PyList_New(total);
    if (!out) goto fail_all;
    Py_ssize_t r = 0;
    for (Py_ssize_t k = 0; k < K; ++k) {
      if (k + 2 < K && pq[k + 2] >= 0 && pq[k + 2] < nd) __builtin_prefetch(PyList_GET_ITEM(docs, pq[k + 2]));
      if (!cnt[k]) continue;
      Py_ssize_t two = 0, ns = 0, nt = 0;
      PyObject **side = pq[k] >= 0 && pq[k] < nd ? seq_items(PyList_GET_ITEM(docs, pq[k]), &two) : NULL;
      PyObject **src = side && two == 2 ? seq_items(side[0], &ns) : NULL;
      PyObject **tgt = side && two == 2 ? seq_items(side[1], &nt) : NULL;
      if (!src || !tgt) {
        PyErr_Format(PyExc_TypeError, "build_rows: docs[%lld] is not a (sentences, sentences) pair", (long long)pq[k]);
        Py_DECREF(out);
        goto fail_all;
      }
      for (int64_t c = 0; c < cnt[k]; ++c, ++r) {
        double score;
        int32_t i, j;
        memcpy(&score, m + 16 * r, 8);
        memcpy(&i, m + 16 * r + 8, 4);
        memcpy(&j, m + 16 * r + 12, 4);
        if (c + 8 < cnt[k]) {  /* the str objects a few rows ahead: their refcounts are the misses here */
          int32_t ia, ja;
          memcpy(&ia, m + 16 * (r + 8) + 8, 4);
          memcpy(&ja, m + 16 * (r + 8) + 12, 4);
          if (ia >= 0 && ia < ns && ja >= 0 && ja < nt) {
            __builtin_prefetch(src[ia], 1);
            __builtin_prefetch(tgt[ja], 1);
          }
        }
        if (i < 0 || j < 0 || i >= ns || j >= nt) {
          PyErr_Format(PyExc_IndexError, "build_rows: match %zd = (%d, %d) outside a %zd x %zd pair", r, i, j, ns, nt);
          Py_DECREF(out);
          goto fail_all;
        }
        PyObject *f = PyFloat_FromDouble(score);
        PyObject *t = f ? PyTuple_New(3) : NULL;
        if (!t) {
          Py_XDECREF(f);
          Py_DECREF(out);
          goto fail_all;
        }
        PyObject *a = src[i], *b = tgt[j];
        Py_INCREF(a);
        Py_INCREF(b);
        PyTuple_SET_ITEM(t, 0, f);
        PyTuple_SET_ITEM(t, 1, a);
        PyTuple_SET_ITEM(t, 2, b);
        /* a float and two str: no cycle possible, so the collector need
           not scan it (CPython untracks such tuples itself, but only when
           a collection gets to them: ~10^5 rows made a 20 ms gen-0 pass) */
        PyObject_GC_UnTrack(t);
        PyList_SET_ITEM(out, r, t);
      }
    }
    PyBuffer_Release(&bm);
    PyBuffer_Release(&bc);
    PyBuffer_Release(&bq);
    return out;
  }
fail_all:
  PyBuffer_Release(&bq);
fail_c:
  PyBuffer_Release(&bc);
fail_m:
  PyBuffer_Release(&bm);
  return NULL;
}

static PyMethodDef methods[] = {
    {"str_view", str_view, METH_VARARGS, "in-place character pointers of a list of compact ASCII str"},
    {"docs_view", docs_view, METH_VARARGS, "in-place character pointers of document pairs' sentences"},
    {"build_rows", build_rows, METH_VARARGS, "(score, source, target) rows of compacted matches"},
    {NULL, NULL, 0, NULL}};

static struct PyModuleDef module = {PyModuleDef_HEAD_INIT, "_pyhost", "CPython helpers of the host path", -1,
                                    methods};

PyMODINIT_FUNC PyInit__pyhost(void) { return PyModule_Create(&module); }
