/* _seqcodec — CPython binding of the host cache calls of include/emm.h.
 *
 * The reference engine calls its cache with a Python list of tuples
 * ("img", content_hash) / ("pfx", prefix_id, i) / ("txt", request_id, i) and
 * a list of int weights (pkg/src/mmsim/engine.py:448-461, cache.py:372-399),
 * tens of thousands of times per trace (scheduler retries, App. A H6).  This
 * module is the binding a maintainer would put between that Python and the C
 * ABI: it walks the list once in C into the injective uint64 keys of keys.py
 * and calls emm_cache_match_prefix / _insert_prefix / _release /
 * _image_lookup / _image_insert through function pointers handed over by the
 * ctypes binding (_lib.py loads libemm.so; this module never links it).
 * Every decision stays in libemm.so (host_cache.cpp).
 *
 * Symbols the C walk does not encode (generic hashables, first sight of an
 * image content hash, out-of-range ids, non-int weights) make the call return
 * None; the caller then takes the Python codec path (keys.py), which also
 * registers the image so the next call is fast.
 */
#define PY_SSIZE_T_CLEAN
#include <Python.h>
#include <stdint.h>
#include <stdlib.h>
#include <structmember.h>

#define NPY_NO_DEPRECATED_API NPY_2_0_API_VERSION
#include <numpy/arrayobject.h>

#define TAG_PFX (1ULL << 62)
#define TAG_TXT (2ULL << 62)

typedef int (*match_fn)(void*, const uint64_t*, const int64_t*, int64_t, double, int64_t*,
                        uint64_t*);
typedef int (*match_lazy_fn)(void*, const uint64_t*, int64_t, int64_t, double, int64_t*,
                             uint64_t*, int32_t*);
typedef int (*insert_fn)(void*, const uint64_t*, const int64_t*, int64_t, double, int64_t*);
typedef int (*release_fn)(void*, uint64_t);
typedef int (*ilookup_fn)(void*, const char*, double, int64_t*);
typedef int (*iinsert_fn)(void*, const char*, int64_t, double, int64_t, int32_t*);

static match_fn f_match;
static match_lazy_fn f_match_lazy;
static insert_fn f_insert;
static release_fn f_release;
static ilookup_fn f_ilookup;
static iinsert_fn f_iinsert;

static PyObject *s_img, *s_pfx, *s_txt, *s_emm_keys, *s_emm_array;
static uint64_t* g_keys;
static int64_t* g_w;
static Py_ssize_t g_cap;

static int reserve(Py_ssize_t n) {
  if (n <= g_cap) return 0;
  Py_ssize_t cap = g_cap ? g_cap : 1024;
  while (cap < n) cap *= 2;
  uint64_t* k = (uint64_t*)realloc(g_keys, (size_t)cap * 8);
  if (!k) return -1;
  g_keys = k;
  int64_t* w = (int64_t*)realloc(g_w, (size_t)cap * 8);
  if (!w) return -1;
  g_w = w;
  g_cap = cap;
  return 0;
}

static PyObject* s_one; /* the small-int singleton 1: the weight of every text symbol */

/* 1 txt, 2 pfx, 3 img, 0 other: interned literals compare by pointer (the
 * engine builds its tuples from literals), anything else by value */
static inline int tag_kind(PyObject* tag) {
  if (tag == s_txt) return 1;
  if (tag == s_pfx) return 2;
  if (tag == s_img) return 3;
  if (PyUnicode_Compare(tag, s_txt) == 0) return 1;
  if (PyUnicode_Compare(tag, s_pfx) == 0) return 2;
  if (PyUnicode_Compare(tag, s_img) == 0) return 3;
  return 0;
}

/* exact int -> long long; 0 when it does not fit */
static inline int as_ll(PyObject* o, long long* v) {
#if PY_VERSION_HEX >= 0x030C0000
  if (PyUnstable_Long_IsCompact((PyLongObject*)o)) {
    *v = (long long)PyUnstable_Long_CompactValue((PyLongObject*)o);
    return 1;
  }
#endif
  int of = 0;
  *v = PyLong_AsLongLongAndOverflow(o, &of);
  return !of && !(*v == -1 && PyErr_Occurred());
}

/* Walk items[start, n) into keys / w.  Returns n, or i when symbol i needs the
 * Python path, or -1 with a Python error set.  Runs of ("txt"|"pfx", id, i)
 * sharing the tag and id objects (as Engine.unified_sequence builds them,
 * engine.py:448-461) reuse the previous symbol's decoded id. */
static Py_ssize_t walk(PyObject** items, PyObject** witems, PyObject* img, uint64_t* keys,
                       int64_t* w, Py_ssize_t start, Py_ssize_t n) {
  Py_ssize_t i = start;
  PyObject *prev_tag = NULL, *prev_id = NULL;
  uint64_t prev_hi = 0;
  for (; i < n; ++i) {
    if (witems) {
      PyObject* wi = witems[i];
      if (wi == s_one) {
        w[i] = 1;
      } else {
        long long v;
        if (!PyLong_CheckExact(wi) || !as_ll(wi, &v)) {
          PyErr_Clear();
          return i;
        }
        w[i] = (int64_t)v;
      }
    } else {
      w[i] = 1;
    }
    PyObject* t = items[i];
    if (!PyTuple_CheckExact(t)) return i;
    Py_ssize_t sz = PyTuple_GET_SIZE(t);
    if (sz < 2) return i;
    PyObject* tag = PyTuple_GET_ITEM(t, 0);
    if (sz == 3) {
      PyObject* a = PyTuple_GET_ITEM(t, 1);
      PyObject* b = PyTuple_GET_ITEM(t, 2);
      long long bv;
      if (!PyLong_CheckExact(b) || !as_ll(b, &bv) || bv < 0 || bv >= (1LL << 32)) {
        PyErr_Clear();
        return i;
      }
      if (tag != prev_tag || a != prev_id) {
        if (!PyUnicode_CheckExact(tag)) return i;
        const int kind = tag_kind(tag);
        if (kind != 1 && kind != 2) return i;
        long long av;
        if (!PyLong_CheckExact(a) || !as_ll(a, &av) || av < 0 || av >= (1LL << 30)) {
          PyErr_Clear();
          return i;
        }
        prev_tag = tag;
        prev_id = a;
        prev_hi = (kind == 1 ? TAG_TXT : TAG_PFX) | ((uint64_t)av << 32);
      }
      keys[i] = prev_hi | (uint64_t)bv;
    } else if (sz == 2 && PyUnicode_CheckExact(tag) && tag_kind(tag) == 3) {
      PyObject* h = PyTuple_GET_ITEM(t, 1);
      if (!PyUnicode_CheckExact(h)) return i;
      PyObject* k = PyDict_GetItemWithError(img, h);
      if (!k) return PyErr_Occurred() ? -1 : i;
      uint64_t kv = PyLong_AsUnsignedLongLong(k);
      if (kv == (uint64_t)-1 && PyErr_Occurred()) return -1;
      keys[i] = kv;
    } else {
      return i;
    }
  }
  return n;
}

/* encode(tokens, weights|None, img_keys, keys_out, w_out, start) -> n | -(i+1) */
static PyObject* encode(PyObject* self, PyObject* args) {
  (void)self;
  PyObject *tokens, *weights, *img;
  Py_buffer kb, wb;
  Py_ssize_t start;
  if (!PyArg_ParseTuple(args, "OOO!w*w*n", &tokens, &weights, &PyDict_Type, &img, &kb, &wb,
                        &start))
    return NULL;
  PyObject *tf = NULL, *wf = NULL, *ret = NULL;
  tf = PySequence_Fast(tokens, "tokens must be a sequence");
  if (!tf) goto done;
  Py_ssize_t n = PySequence_Fast_GET_SIZE(tf);
  if (weights != Py_None) {
    wf = PySequence_Fast(weights, "weights must be a sequence");
    if (!wf) goto done;
    Py_ssize_t nw = PySequence_Fast_GET_SIZE(wf);
    if (nw < n) n = nw;
  }
  if ((Py_ssize_t)(kb.len / 8) < n || (Py_ssize_t)(wb.len / 8) < n) {
    PyErr_SetString(PyExc_ValueError, "output buffers too small");
    goto done;
  }
  Py_ssize_t r = walk(PySequence_Fast_ITEMS(tf), wf ? PySequence_Fast_ITEMS(wf) : NULL, img,
                      (uint64_t*)kb.buf, (int64_t*)wb.buf, start < 0 ? 0 : start, n);
  if (r < 0) goto done;
  ret = PyLong_FromSsize_t(r < n ? -(r + 1) : n);
done:
  Py_XDECREF(tf);
  Py_XDECREF(wf);
  PyBuffer_Release(&kb);
  PyBuffer_Release(&wb);
  return ret;
}

/* Resolve (tokens, weights) to key / weight pointers.  Returns 1 on success,
 * 0 when the Python path must handle the call, -1 on error.  Buffers held in
 * kb / wb (released by seq_release). */
typedef struct {
  const uint64_t* keys;
  const int64_t* w;
  int64_t n;
  Py_buffer kb, wb;
  int hk, hw;
} seq_t;

/* hk / hw: 1 = a Py_buffer to release, 2 = a plain reference to the ndarray
 * whose data pointer is used directly (kb.obj / wb.obj) */
static void seq_release(seq_t* s) {
  if (s->hk == 1) PyBuffer_Release(&s->kb);
  if (s->hk == 2) Py_DECREF(s->kb.obj);
  if (s->hw == 1) PyBuffer_Release(&s->wb);
  if (s->hw == 2) Py_DECREF(s->wb.obj);
}

/* Returns 1 (buffer held) or 2 (ndarray fast path: numpy's buffer export
 * formats a descriptor string per call, ~0.3 us, more than the tree walk),
 * -1 on error. */
static int get_u64_buffer(PyObject* o, Py_buffer* b) {
  if (PyArray_CheckExact(o)) {
    PyArrayObject* a = (PyArrayObject*)o;
    if (PyArray_ITEMSIZE(a) == 8 && PyArray_IS_C_CONTIGUOUS(a)) {
      Py_INCREF(o);
      b->obj = o;
      b->buf = PyArray_DATA(a);
      b->len = (Py_ssize_t)PyArray_SIZE(a) * 8;
      b->itemsize = 8;
      return 2;
    }
  }
  if (PyObject_GetBuffer(o, b, PyBUF_C_CONTIGUOUS | PyBUF_FORMAT) < 0) return -1;
  if (b->itemsize != 8) {
    PyBuffer_Release(b);
    PyErr_SetString(PyExc_TypeError, "expected an 8-byte element buffer");
    return -1;
  }
  return 1;
}

static int resolve(PyObject* tokens, PyObject* weights, PyObject* img, seq_t* s) {
  s->hk = s->hw = 0;
  PyObject* pre = NULL;
  if (!PyList_CheckExact(tokens) && !PyTuple_CheckExact(tokens)) {
    pre = PyObject_GetAttr(tokens, s_emm_keys);
    if (!pre) {
      if (!PyErr_ExceptionMatches(PyExc_AttributeError)) return -1;
      PyErr_Clear();
    }
  }
  if (pre) {  /* precomputed keys (keys.SymbolSeq / KeySeq) */
    PyObject* prew = NULL;
    if (weights != Py_None) {
      prew = PyObject_GetAttr(weights, s_emm_array);
      if (!prew) {
        Py_DECREF(pre);
        if (!PyErr_ExceptionMatches(PyExc_AttributeError)) return -1;
        PyErr_Clear();
        return 0;
      }
    }
    int rc = get_u64_buffer(pre, &s->kb);
    Py_DECREF(pre);
    if (rc < 0) {
      Py_XDECREF(prew);
      return -1;
    }
    s->hk = rc;
    s->keys = (const uint64_t*)s->kb.buf;
    s->n = s->kb.len / 8;
    if (prew) {
      rc = get_u64_buffer(prew, &s->wb);
      Py_DECREF(prew);
      if (rc < 0) return -1;
      s->hw = rc;
      s->w = (const int64_t*)s->wb.buf;
      if (s->wb.len / 8 < s->n) s->n = s->wb.len / 8;
    } else {
      if (reserve(s->n) < 0) {
        PyErr_NoMemory();
        return -1;
      }
      for (int64_t i = 0; i < s->n; ++i) g_w[i] = 1;
      s->w = g_w;
    }
    return 1;
  }
  if (!PyList_Check(tokens) && !PyTuple_Check(tokens)) return 0;
  PyObject** items = PySequence_Fast_ITEMS(tokens);
  Py_ssize_t n = PySequence_Fast_GET_SIZE(tokens);
  PyObject** witems = NULL;
  if (weights != Py_None) {
    if (!PyList_Check(weights) && !PyTuple_Check(weights)) return 0;
    Py_ssize_t nw = PySequence_Fast_GET_SIZE(weights);
    if (nw < n) n = nw;
    witems = PySequence_Fast_ITEMS(weights);
  }
  if (reserve(n) < 0) {
    PyErr_NoMemory();
    return -1;
  }
  Py_ssize_t r = walk(items, witems, img, g_keys, g_w, 0, n);
  if (r < 0) return -1;
  if (r < n) return 0;
  s->keys = g_keys;
  s->w = g_w;
  s->n = n;
  return 1;
}

static void* as_ptr(PyObject* o) { return PyLong_AsVoidPtr(o); }

/* match(cache, tokens, weights, img_keys, now) -> (rc, matched, handle) | None
 * The reference walk stops at the first mismatch (cache.py:121-156), so a
 * symbol list is encoded lazily: a first chunk, then 4x more only while the
 * tree walk runs past what is encoded (emm_cache_match_prefix_lazy). */
static PyObject* match(PyObject* self, PyObject* args) {
  (void)self;
  PyObject *cp, *tokens, *weights, *img;
  double now;
  if (!PyArg_ParseTuple(args, "OOOO!d", &cp, &tokens, &weights, &PyDict_Type, &img, &now))
    return NULL;
  void* c = as_ptr(cp);
  if (!c && PyErr_Occurred()) return NULL;
  int64_t m = 0;
  uint64_t h = 0;
  int32_t more = 0;
  int rc;
  if (PyList_Check(tokens) || PyTuple_Check(tokens)) {
    PyObject* pre = NULL;
    if (!PyList_CheckExact(tokens) && !PyTuple_CheckExact(tokens)) {
      pre = PyObject_GetAttr(tokens, s_emm_keys);
      if (!pre) {
        if (!PyErr_ExceptionMatches(PyExc_AttributeError)) return NULL;
        PyErr_Clear();
      }
    }
    if (!pre) {
      PyObject** items = PySequence_Fast_ITEMS(tokens);
      Py_ssize_t n = PySequence_Fast_GET_SIZE(tokens);
      PyObject** witems = NULL;
      if (weights != Py_None) {
        if (!PyList_Check(weights) && !PyTuple_Check(weights)) Py_RETURN_NONE;
        Py_ssize_t nw = PySequence_Fast_GET_SIZE(weights);
        if (nw < n) n = nw;
        witems = PySequence_Fast_ITEMS(weights);
      }
      if (reserve(n) < 0) return PyErr_NoMemory();
      Py_ssize_t avail = 0, target = n < 1 ? n : 1;
      for (;;) {
        Py_ssize_t r = walk(items, witems, img, g_keys, g_w, avail, target);
        if (r < 0) return NULL;
        if (r < target) Py_RETURN_NONE;
        rc = f_match_lazy(c, g_keys, target, n, now, &m, &h, &more);
        if (rc || !more) break;
        avail = target;
        target = target < 32 ? 32 : target * 4;
        if (target > n) target = n;
      }
      return Py_BuildValue("iLK", rc, (long long)m, (unsigned long long)h);
    }
    Py_DECREF(pre);
  }
  seq_t s;
  int r = resolve(tokens, weights, img, &s);
  if (r < 0) return NULL;
  if (r == 0) Py_RETURN_NONE;
  rc = f_match(c, s.keys, s.w, s.n, now, &m, &h);
  seq_release(&s);
  return Py_BuildValue("iLK", rc, (long long)m, (unsigned long long)h);
}

/* insert(cache, tokens, weights, img_keys, now) -> (rc, added) | None */
static PyObject* insert(PyObject* self, PyObject* args) {
  (void)self;
  PyObject *cp, *tokens, *weights, *img;
  double now;
  if (!PyArg_ParseTuple(args, "OOOO!d", &cp, &tokens, &weights, &PyDict_Type, &img, &now))
    return NULL;
  void* c = as_ptr(cp);
  if (!c && PyErr_Occurred()) return NULL;
  seq_t s;
  int r = resolve(tokens, weights, img, &s);
  if (r < 0) return NULL;
  if (r == 0) Py_RETURN_NONE;
  int64_t added = 0;
  int rc = f_insert(c, s.keys, s.w, s.n, now, &added);
  seq_release(&s);
  return Py_BuildValue("iL", rc, (long long)added);
}

static PyObject* release(PyObject* self, PyObject* args) {
  (void)self;
  PyObject* cp;
  unsigned long long h;
  if (!PyArg_ParseTuple(args, "OK", &cp, &h)) return NULL;
  void* c = as_ptr(cp);
  if (!c && PyErr_Occurred()) return NULL;
  return PyLong_FromLong(f_release(c, (uint64_t)h));
}

static PyObject* image_lookup(PyObject* self, PyObject* args) {
  (void)self;
  PyObject* cp;
  const char* hs;
  double now;
  if (!PyArg_ParseTuple(args, "Osd", &cp, &hs, &now)) return NULL;
  void* c = as_ptr(cp);
  if (!c && PyErr_Occurred()) return NULL;
  int64_t out = -1;
  int rc = f_ilookup(c, hs, now, &out);
  return Py_BuildValue("iL", rc, (long long)out);
}

static PyObject* image_insert(PyObject* self, PyObject* args) {
  (void)self;
  PyObject* cp;
  const char* hs;
  long long tok, nbytes;
  double now;
  if (!PyArg_ParseTuple(args, "OsLdL", &cp, &hs, &tok, &now, &nbytes)) return NULL;
  void* c = as_ptr(cp);
  if (!c && PyErr_Occurred()) return NULL;
  int32_t ok = 0;
  int rc = f_iinsert(c, hs, (int64_t)tok, now, (int64_t)nbytes, &ok);
  return Py_BuildValue("ii", rc, (int)ok);
}

/* bind(match, match_lazy, insert, release, image_lookup, image_insert) */
static PyObject* bind(PyObject* self, PyObject* args) {
  (void)self;
  PyObject *a, *al, *b, *c, *d, *e;
  if (!PyArg_ParseTuple(args, "OOOOOO", &a, &al, &b, &c, &d, &e)) return NULL;
  f_match = (match_fn)PyLong_AsVoidPtr(a);
  f_match_lazy = (match_lazy_fn)PyLong_AsVoidPtr(al);
  f_insert = (insert_fn)PyLong_AsVoidPtr(b);
  f_release = (release_fn)PyLong_AsVoidPtr(c);
  f_ilookup = (ilookup_fn)PyLong_AsVoidPtr(d);
  f_iinsert = (iinsert_fn)PyLong_AsVoidPtr(e);
  if (PyErr_Occurred()) return NULL;
  if (!f_match || !f_match_lazy || !f_insert || !f_release || !f_ilookup || !f_iinsert) {
    PyErr_SetString(PyExc_ValueError, "null entry point");
    return NULL;
  }
  Py_RETURN_NONE;
}


/* ------------------------------------------------------------------ types
 * Handle  — the match handle (cache.py:93-103): id, owning tree, released.
 *           cache.MatchHandle subclasses it (adds `entries`).
 * Core    — base class of cache.GpuUnifiedCache: match_prefix, insert_prefix,
 *           release and image_lookup as C methods (METH_FASTCALL), so the
 *           reference engine's tens of thousands of calls per trace pay a C
 *           call each instead of a Python method + argument tuple + handle
 *           __init__.  Sequences the C walk cannot encode fall back to the
 *           subclass's Python _match_slow / _insert_slow; nonzero C-ABI codes
 *           go through the subclass's _raise (the _lib.check mapping). */
typedef struct {
  PyObject_HEAD
  unsigned long long id;
  PyObject* tree;
  char released;
} HandleObject;

static int handle_init(HandleObject* self, PyObject* args, PyObject* kw) {
  (void)kw;
  unsigned long long id;
  PyObject* tree;
  if (!PyArg_ParseTuple(args, "KO", &id, &tree)) return -1;
  self->id = id;
  Py_INCREF(tree);
  Py_XSETREF(self->tree, tree);
  self->released = 0;
  return 0;
}

static int handle_traverse(HandleObject* self, visitproc visit, void* arg) {
  Py_VISIT(self->tree);
  return 0;
}

static int handle_clear(HandleObject* self) {
  Py_CLEAR(self->tree);
  return 0;
}

static void handle_dealloc(HandleObject* self) {
  PyTypeObject* tp = Py_TYPE(self);
  PyObject_GC_UnTrack(self);
  handle_clear(self);
  tp->tp_free((PyObject*)self);  /* subtype_dealloc drops the heap subtype's reference */
}

static PyMemberDef handle_members[] = {
    {"_id", T_ULONGLONG, offsetof(HandleObject, id), 0, "handle id"},
    {"_tree", T_OBJECT, offsetof(HandleObject, tree), 0, "owning tree"},
    {"released", T_BOOL, offsetof(HandleObject, released), 0, "released once"},
    {NULL, 0, 0, 0, NULL}};

static PyTypeObject HandleType = {
    PyVarObject_HEAD_INIT(NULL, 0).tp_name = "_seqcodec.Handle",
    .tp_basicsize = sizeof(HandleObject),
    .tp_flags = Py_TPFLAGS_DEFAULT | Py_TPFLAGS_BASETYPE | Py_TPFLAGS_HAVE_GC,
    .tp_new = PyType_GenericNew,
    .tp_init = (initproc)handle_init,
    .tp_dealloc = (destructor)handle_dealloc,
    .tp_traverse = (traverseproc)handle_traverse,
    .tp_clear = (inquiry)handle_clear,
    .tp_members = handle_members,
};

typedef struct {
  PyObject_HEAD
  void* cache;
  PyObject* img;      /* codec._img_key */
  PyObject* tree;     /* PrefixTree: the handles' owner */
  PyObject* htype;    /* MatchHandle (a Handle subclass) */
  PyObject* release_error;
} CoreObject;

static PyObject *s_match_slow, *s_insert_slow, *s_raise;

/* positional or keyword arguments of a METH_FASTCALL | METH_KEYWORDS method
 * into out[0..n) by the reference's parameter names (cache.py:372-406) */
static int bind_args(const char* fn, PyObject* const* args, Py_ssize_t nargs, PyObject* kwnames,
                     const char* const* names, int n, PyObject** out) {
  if (nargs > n) {
    PyErr_Format(PyExc_TypeError, "%s() takes %d arguments (%zd given)", fn, n, nargs);
    return -1;
  }
  for (int i = 0; i < n; ++i) out[i] = i < nargs ? args[i] : NULL;
  Py_ssize_t nk = kwnames ? PyTuple_GET_SIZE(kwnames) : 0;
  for (Py_ssize_t j = 0; j < nk; ++j) {
    PyObject* key = PyTuple_GET_ITEM(kwnames, j);
    int hit = -1;
    for (int i = 0; i < n; ++i)
      if (PyUnicode_CompareWithASCIIString(key, names[i]) == 0) hit = i;
    if (hit < 0 || out[hit]) {
      PyErr_Format(PyExc_TypeError, "%s() got an unexpected or repeated argument %R", fn, key);
      return -1;
    }
    out[hit] = args[nargs + j];
  }
  for (int i = 0; i < n; ++i)
    if (!out[i]) {
      PyErr_Format(PyExc_TypeError, "%s() missing argument '%s'", fn, names[i]);
      return -1;
    }
  return 0;
}

static const char* const kw_seq[] = {"tokens", "weights", "now"};
static const char* const kw_img[] = {"content_hash", "now"};
static const char* const kw_rel[] = {"handle"};

static int core_traverse(CoreObject* self, visitproc visit, void* arg) {
  Py_VISIT(self->img);
  Py_VISIT(self->tree);
  Py_VISIT(self->htype);
  Py_VISIT(self->release_error);
  return 0;
}

static int core_clear(CoreObject* self) {
  Py_CLEAR(self->img);
  Py_CLEAR(self->tree);
  Py_CLEAR(self->htype);
  Py_CLEAR(self->release_error);
  return 0;
}

static void core_dealloc(CoreObject* self) {
  PyTypeObject* tp = Py_TYPE(self);
  PyObject_GC_UnTrack(self);
  core_clear(self);
  tp->tp_free((PyObject*)self);  /* subtype_dealloc drops the heap subtype's reference */
}

/* _core_bind(cache_ptr, img_keys, tree, handle_type, release_error) */
static PyObject* core_bind(CoreObject* self, PyObject* const* a, Py_ssize_t n) {
  if (n != 5 || !PyDict_Check(a[1]) || !PyType_Check(a[3]) ||
      !PyType_IsSubtype((PyTypeObject*)a[3], &HandleType)) {
    PyErr_SetString(PyExc_TypeError, "_core_bind(cache, img_keys, tree, handle_type, error)");
    return NULL;
  }
  void* c = PyLong_AsVoidPtr(a[0]);
  if (!c && PyErr_Occurred()) return NULL;
  self->cache = c;
  Py_INCREF(a[1]);
  Py_XSETREF(self->img, a[1]);
  Py_INCREF(a[2]);
  Py_XSETREF(self->tree, a[2]);
  Py_INCREF(a[3]);
  Py_XSETREF(self->htype, a[3]);
  Py_INCREF(a[4]);
  Py_XSETREF(self->release_error, a[4]);
  Py_RETURN_NONE;
}

static PyObject* core_unbind(CoreObject* self, PyObject* unused) {
  (void)unused;
  self->cache = NULL;
  Py_RETURN_NONE;
}

static int core_ready(CoreObject* self) {
  if (!self->cache || !self->htype) {
    PyErr_SetString(PyExc_RuntimeError, "cache core is not bound (or already destroyed)");
    return 0;
  }
  return 1;
}

static PyObject* core_raise(CoreObject* self, int rc) {
  PyObject* r = PyObject_CallMethodOneArg((PyObject*)self, s_raise, PyLong_FromLong(rc));
  Py_XDECREF(r);
  if (!PyErr_Occurred()) PyErr_Format(PyExc_RuntimeError, "emm error %d", rc);
  return NULL;
}

static PyObject* new_handle(CoreObject* self, uint64_t hid) {
  PyTypeObject* tp = (PyTypeObject*)self->htype;
  HandleObject* h = (HandleObject*)tp->tp_alloc(tp, 0);
  if (!h) return NULL;
  h->id = hid;
  Py_INCREF(self->tree);
  h->tree = self->tree;
  h->released = 0;
  return (PyObject*)h;
}

static int parse_now(PyObject* o, double* now) {
  *now = PyFloat_AsDouble(o);
  return !(*now == -1.0 && PyErr_Occurred());
}

/* match_prefix(tokens, weights, now) -> (matched, handle)   cache.py:372-383 */
static PyObject* core_match(CoreObject* self, PyObject* const* args, Py_ssize_t nargs,
                            PyObject* kwnames) {
  PyObject* a[3];
  if (bind_args("match_prefix", args, nargs, kwnames, kw_seq, 3, a) < 0) return NULL;
  if (!core_ready(self)) return NULL;
  PyObject *tokens = a[0], *weights = a[1];
  double now;
  if (!parse_now(a[2], &now)) return NULL;
  int64_t m = 0;
  uint64_t h = 0;
  int32_t more = 0;
  int rc = 0, done = 0;
  if (PyList_CheckExact(tokens) || PyTuple_CheckExact(tokens)) {
    PyObject** items = PySequence_Fast_ITEMS(tokens);
    Py_ssize_t len = PySequence_Fast_GET_SIZE(tokens);
    PyObject** witems = NULL;
    int ok = 1;
    if (weights != Py_None) {
      if (PyList_Check(weights) || PyTuple_Check(weights)) {
        Py_ssize_t nw = PySequence_Fast_GET_SIZE(weights);
        if (nw < len) len = nw;
        witems = PySequence_Fast_ITEMS(weights);
      } else {
        ok = 0;
      }
    }
    if (ok) {
      if (reserve(len) < 0) return PyErr_NoMemory();
      Py_ssize_t avail = 0, target = len < 1 ? len : 1;
      for (;;) {
        Py_ssize_t r = walk(items, witems, self->img, g_keys, g_w, avail, target);
        if (r < 0) return NULL;
        if (r < target) break;  /* needs the Python codec */
        rc = f_match_lazy(self->cache, g_keys, target, len, now, &m, &h, &more);
        if (rc || !more) {
          done = 1;
          break;
        }
        avail = target;
        target = target < 32 ? 32 : target * 4;
        if (target > len) target = len;
      }
    }
  } else {
    seq_t s;
    int r = resolve(tokens, weights, self->img, &s);
    if (r < 0) return NULL;
    if (r > 0) {
      rc = f_match(self->cache, s.keys, s.w, s.n, now, &m, &h);
      seq_release(&s);
      done = 1;
    }
  }
  if (!done) return PyObject_VectorcallMethod(s_match_slow, (PyObject* const[]){(PyObject*)self,
                                              tokens, weights, a[2]}, 4, NULL);
  if (rc) return core_raise(self, rc);
  PyObject* hd = new_handle(self, h);
  if (!hd) return NULL;
  PyObject* mm = PyLong_FromLongLong(m);
  if (!mm) {
    Py_DECREF(hd);
    return NULL;
  }
  PyObject* t = PyTuple_New(2);
  if (!t) {
    Py_DECREF(mm);
    Py_DECREF(hd);
    return NULL;
  }
  PyTuple_SET_ITEM(t, 0, mm);
  PyTuple_SET_ITEM(t, 1, hd);
  return t;
}

/* insert_prefix(tokens, weights, now) -> added tokens   cache.py:385-396 */
static PyObject* core_insert(CoreObject* self, PyObject* const* args, Py_ssize_t nargs,
                             PyObject* kwnames) {
  PyObject* a[3];
  if (bind_args("insert_prefix", args, nargs, kwnames, kw_seq, 3, a) < 0) return NULL;
  if (!core_ready(self)) return NULL;
  double now;
  if (!parse_now(a[2], &now)) return NULL;
  seq_t s;
  int r = resolve(a[0], a[1], self->img, &s);
  if (r < 0) return NULL;
  if (r == 0)
    return PyObject_VectorcallMethod(s_insert_slow, (PyObject* const[]){(PyObject*)self, a[0],
                                     a[1], a[2]}, 4, NULL);
  int64_t added = 0;
  int rc = f_insert(self->cache, s.keys, s.w, s.n, now, &added);
  seq_release(&s);
  if (rc) return core_raise(self, rc);
  return PyLong_FromLongLong(added);
}

/* release(handle)   cache.py:398-406 */
static PyObject* core_release(CoreObject* self, PyObject* const* args, Py_ssize_t nargs,
                              PyObject* kwnames) {
  PyObject* handle;
  if (bind_args("release", args, nargs, kwnames, kw_rel, 1, &handle) < 0) return NULL;
  if (!core_ready(self)) return NULL;
  if (!PyObject_TypeCheck(handle, &HandleType) || ((HandleObject*)handle)->tree != self->tree ||
      ((HandleObject*)handle)->released) {
    PyErr_SetString(self->release_error, "handle already released or unknown");
    return NULL;
  }
  int rc = f_release(self->cache, (uint64_t)((HandleObject*)handle)->id);
  if (rc) return core_raise(self, rc);
  ((HandleObject*)handle)->released = 1;
  Py_RETURN_NONE;
}

/* image_lookup(content_hash, now) -> token_count | None   cache.py:372-376 */
static PyObject* core_image_lookup(CoreObject* self, PyObject* const* args, Py_ssize_t nargs,
                                   PyObject* kwnames) {
  PyObject* a[2];
  if (bind_args("image_lookup", args, nargs, kwnames, kw_img, 2, a) < 0) return NULL;
  if (!PyUnicode_Check(a[0])) {
    PyErr_SetString(PyExc_TypeError, "image_lookup(content_hash: str, now)");
    return NULL;
  }
  if (!core_ready(self)) return NULL;
  double now;
  if (!parse_now(a[1], &now)) return NULL;
  const char* hs = PyUnicode_AsUTF8(a[0]);
  if (!hs) return NULL;
  int64_t out = -1;
  int rc = f_ilookup(self->cache, hs, now, &out);
  if (rc) return core_raise(self, rc);
  if (out < 0) Py_RETURN_NONE;
  return PyLong_FromLongLong(out);
}

static PyMethodDef core_methods[] = {
    {"_core_bind", (PyCFunction)(void (*)(void))core_bind, METH_FASTCALL, NULL},
    {"_core_unbind", (PyCFunction)core_unbind, METH_NOARGS, NULL},
    {"match_prefix", (PyCFunction)(void (*)(void))core_match, METH_FASTCALL | METH_KEYWORDS,
     "match_prefix(tokens, weights, now) -> (matched_tokens, handle)"},
    {"insert_prefix", (PyCFunction)(void (*)(void))core_insert, METH_FASTCALL | METH_KEYWORDS,
     "insert_prefix(tokens, weights, now) -> inserted tokens"},
    {"release", (PyCFunction)(void (*)(void))core_release, METH_FASTCALL | METH_KEYWORDS,
     "release(handle)"},
    {"image_lookup", (PyCFunction)(void (*)(void))core_image_lookup,
     METH_FASTCALL | METH_KEYWORDS, "image_lookup(content_hash, now) -> token_count | None"},
    {NULL, NULL, 0, NULL}};

static PyTypeObject CoreType = {
    PyVarObject_HEAD_INIT(NULL, 0).tp_name = "_seqcodec.Core",
    .tp_basicsize = sizeof(CoreObject),
    .tp_flags = Py_TPFLAGS_DEFAULT | Py_TPFLAGS_BASETYPE | Py_TPFLAGS_HAVE_GC,
    .tp_new = PyType_GenericNew,
    .tp_dealloc = (destructor)core_dealloc,
    .tp_traverse = (traverseproc)core_traverse,
    .tp_clear = (inquiry)core_clear,
    .tp_methods = core_methods,
};

static PyMethodDef methods[] = {
    {"encode", encode, METH_VARARGS, "encode(tokens, weights, img_keys, keys_out, w_out, start)"},
    {"bind", bind, METH_VARARGS, "bind(match, match_lazy, insert, release, image_lookup, image_insert)"},
    {"match", match, METH_VARARGS, "match(cache, tokens, weights, img_keys, now)"},
    {"insert", insert, METH_VARARGS, "insert(cache, tokens, weights, img_keys, now)"},
    {"release", release, METH_VARARGS, "release(cache, handle) -> rc"},
    {"image_lookup", image_lookup, METH_VARARGS, "image_lookup(cache, hash, now)"},
    {"image_insert", image_insert, METH_VARARGS, "image_insert(cache, hash, tokens, now, bytes)"},
    {NULL, NULL, 0, NULL}};

static struct PyModuleDef mod = {PyModuleDef_HEAD_INIT, "_seqcodec", NULL, -1, methods,
                                 NULL, NULL, NULL, NULL};

PyMODINIT_FUNC PyInit__seqcodec(void) {
  import_array();
  s_img = PyUnicode_InternFromString("img");
  s_pfx = PyUnicode_InternFromString("pfx");
  s_txt = PyUnicode_InternFromString("txt");
  s_emm_keys = PyUnicode_InternFromString("emm_keys");
  s_emm_array = PyUnicode_InternFromString("emm_array");
  s_one = PyLong_FromLong(1);
  s_match_slow = PyUnicode_InternFromString("_match_slow");
  s_insert_slow = PyUnicode_InternFromString("_insert_slow");
  s_raise = PyUnicode_InternFromString("_raise");
  if (!s_img || !s_pfx || !s_txt || !s_emm_keys || !s_emm_array || !s_match_slow ||
      !s_insert_slow || !s_raise || !s_one)
    return NULL;
  if (PyType_Ready(&HandleType) < 0 || PyType_Ready(&CoreType) < 0) return NULL;
  PyObject* m = PyModule_Create(&mod);
  if (!m) return NULL;
  Py_INCREF(&HandleType);
  Py_INCREF(&CoreType);
  if (PyModule_AddObject(m, "Handle", (PyObject*)&HandleType) < 0 ||
      PyModule_AddObject(m, "Core", (PyObject*)&CoreType) < 0) {
    Py_DECREF(m);
    return NULL;
  }
  return m;
}
