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
 *   build_rows(matches, counts, src_first, tgt_first, sentences) -> list
 *       The mining rows (score, source sentence, target sentence) of
 *       align.py:441-447, in pair order: pair k owns the next counts[k]
 *       records of `matches` (bimine_match: f64 score, i32 i, i32 j), whose
 *       sentences are sentences[src_first[k] + i] and
 *       sentences[tgt_first[k] + j].
 */
#define PY_SSIZE_T_CLEAN
#include <Python.h>
#include <stdint.h>
#include <string.h>

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

static PyObject *build_rows(PyObject *self, PyObject *args) {
  PyObject *mo, *co, *so, *to, *list;
  if (!PyArg_ParseTuple(args, "OOOOO!", &mo, &co, &so, &to, &PyList_Type, &list)) return NULL;
  Py_buffer bm, bc, bs, bt;
  if (get_buf(mo, &bm, 0, 16, "matches") < 0) return NULL;
  if (get_buf(co, &bc, 0, 8, "counts") < 0) goto fail_m;
  if (get_buf(so, &bs, 0, 8, "src_first") < 0) goto fail_c;
  if (get_buf(to, &bt, 0, 8, "tgt_first") < 0) goto fail_s;
  {
    const Py_ssize_t K = bc.len / 8, total = bm.len / 16, ns = PyList_GET_SIZE(list);
    const int64_t *cnt = (const int64_t *)bc.buf, *sf = (const int64_t *)bs.buf, *tf = (const int64_t *)bt.buf;
    const char *m = (const char *)bm.buf;
    if (bs.len / 8 != K || bt.len / 8 != K) {
      PyErr_SetString(PyExc_ValueError, "build_rows: counts, src_first and tgt_first differ in length");
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
      for (int64_t c = 0; c < cnt[k]; ++c, ++r) {
        double score;
        int32_t i, j;
        memcpy(&score, m + 16 * r, 8);
        memcpy(&i, m + 16 * r + 8, 4);
        memcpy(&j, m + 16 * r + 12, 4);
        const int64_t si = sf[k] + i, ti = tf[k] + j;
        if (i < 0 || j < 0 || si >= ns || ti >= ns) {
          PyErr_Format(PyExc_IndexError, "build_rows: match %zd refers to sentence %lld / %lld of %zd", r,
                       (long long)si, (long long)ti, ns);
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
        PyObject *a = PyList_GET_ITEM(list, si), *b = PyList_GET_ITEM(list, ti);
        Py_INCREF(a);
        Py_INCREF(b);
        PyTuple_SET_ITEM(t, 0, f);
        PyTuple_SET_ITEM(t, 1, a);
        PyTuple_SET_ITEM(t, 2, b);
        PyList_SET_ITEM(out, r, t);
      }
    }
    PyBuffer_Release(&bm);
    PyBuffer_Release(&bc);
    PyBuffer_Release(&bs);
    PyBuffer_Release(&bt);
    return out;
  }
fail_all:
  PyBuffer_Release(&bt);
fail_s:
  PyBuffer_Release(&bs);
fail_c:
  PyBuffer_Release(&bc);
fail_m:
  PyBuffer_Release(&bm);
  return NULL;
}

static PyMethodDef methods[] = {
    {"str_view", str_view, METH_VARARGS, "in-place character pointers of a list of compact ASCII str"},
    {"build_rows", build_rows, METH_VARARGS, "(score, source, target) rows of compacted matches"},
    {NULL, NULL, 0, NULL}};

static struct PyModuleDef module = {PyModuleDef_HEAD_INIT, "_pyhost", "CPython helpers of the host path", -1,
                                    methods};

PyMODINIT_FUNC PyInit__pyhost(void) { return PyModule_Create(&module); }
