/* wd_host.c -- host side of the drop-in boundary (CPython extension _wdhost).
 *
 * The reference's kernel API takes the corpus as a list of per-document word
 * arrays and returns z the same way (kernels.py:364-377 _gather_words,
 * _ragged_zeros; kernels.py:487-539).  At configs[2]-[4] sizes (1e6 documents)
 * the per-document Python work around the device draw -- building the CSR
 * word array, checking the cached upload still matches, and creating one
 * output array per document -- cost more than the draw itself.  These loops
 * run here in C:
 *
 *   ragged_views(z, offsets)        -> list of 1-D views z[offsets[m]:offsets[m+1]]
 *                                      (one buffer, the views keep it alive)
 *   list_ids(lst)                   -> int64 array of the element object ids
 *   ids_equal(lst, ids)             -> bool: same length, same element objects
 *   concat_ragged(lst, lengths)     -> (int32 words[sum lengths], min, max):
 *                                      element m contributes its first
 *                                      lengths[m] entries (int64 / int32 /
 *                                      int16 / uint16 / uint8 ndarrays); raises
 *                                      TypeError for anything else (the caller
 *                                      then uses numpy), ValueError when a list
 *                                      is shorter than its length, OverflowError
 *                                      when an id does not fit int32.
 *   widen_i32(addr, n, threads)     -> fresh int64 array of the n int32 at addr
 *                                      (e.g. a pinned D2H buffer): an anonymous
 *                                      mapping advised for transparent huge
 *                                      pages, filled by `threads` threads
 *                                      (the page faults of a fresh 1.6 GB
 *                                      buffer cost more than the copy).
 */
#define PY_SSIZE_T_CLEAN
#include <Python.h>
#define NPY_NO_DEPRECATED_API NPY_1_7_API_VERSION
#include <numpy/arrayobject.h>
#include <pthread.h>
#include <stdint.h>
#include <string.h>
#include <sys/mman.h>
#include <unistd.h>

static PyObject* ragged_views(PyObject* self, PyObject* args) {
  PyArrayObject *z, *off;
  (void)self;
  if (!PyArg_ParseTuple(args, "O!O!", &PyArray_Type, &z, &PyArray_Type, &off)) return NULL;
  if (PyArray_NDIM(z) != 1 || PyArray_NDIM(off) != 1 || PyArray_TYPE(off) != NPY_INT64 ||
      !PyArray_ISCARRAY_RO(z) || !PyArray_ISCARRAY_RO(off)) {
    PyErr_SetString(PyExc_ValueError, "ragged_views: need 1-D contiguous z and int64 offsets");
    return NULL;
  }
  const npy_int64* o = (const npy_int64*)PyArray_DATA(off);
  npy_intp m = PyArray_DIM(off, 0) - 1;
  const npy_intp n = PyArray_DIM(z, 0);
  if (m < 0) m = 0;
  PyObject* out = PyList_New(m);
  if (!out) return NULL;
  PyArray_Descr* d = PyArray_DESCR(z);
  char* base = PyArray_BYTES(z);
  const npy_intp isz = PyArray_ITEMSIZE(z);
  const int flags = PyArray_FLAGS(z) & (NPY_ARRAY_WRITEABLE | NPY_ARRAY_C_CONTIGUOUS | NPY_ARRAY_ALIGNED);
  for (npy_intp i = 0; i < m; ++i) {
    const npy_intp a = (npy_intp)o[i], b = (npy_intp)o[i + 1];
    if (a < 0 || b < a || b > n) {
      Py_DECREF(out);
      PyErr_SetString(PyExc_ValueError, "ragged_views: offsets out of range");
      return NULL;
    }
    npy_intp len = b - a;
    Py_INCREF(d);
    PyObject* v = PyArray_NewFromDescr(&PyArray_Type, d, 1, &len, NULL, base + a * isz, flags, NULL);
    if (!v) {
      Py_DECREF(out);
      return NULL;
    }
    Py_INCREF(z);
    if (PyArray_SetBaseObject((PyArrayObject*)v, (PyObject*)z) < 0) {
      Py_DECREF(v);
      Py_DECREF(out);
      return NULL;
    }
    PyList_SET_ITEM(out, i, v);
  }
  return out;
}

static PyObject* list_ids(PyObject* self, PyObject* lst) {
  (void)self;
  if (!PyList_Check(lst)) {
    PyErr_SetString(PyExc_TypeError, "list_ids: need a list");
    return NULL;
  }
  npy_intp m = PyList_GET_SIZE(lst);
  PyObject* out = PyArray_SimpleNew(1, &m, NPY_INT64);
  if (!out) return NULL;
  npy_int64* p = (npy_int64*)PyArray_DATA((PyArrayObject*)out);
  for (npy_intp i = 0; i < m; ++i) p[i] = (npy_int64)(intptr_t)PyList_GET_ITEM(lst, i);
  return out;
}

static PyObject* ids_equal(PyObject* self, PyObject* args) {
  PyObject* lst;
  PyArrayObject* ids;
  (void)self;
  if (!PyArg_ParseTuple(args, "O!O!", &PyList_Type, &lst, &PyArray_Type, &ids)) return NULL;
  if (PyArray_NDIM(ids) != 1 || PyArray_TYPE(ids) != NPY_INT64 || !PyArray_ISCARRAY_RO(ids)) {
    PyErr_SetString(PyExc_ValueError, "ids_equal: need 1-D int64 ids");
    return NULL;
  }
  const npy_intp m = PyList_GET_SIZE(lst);
  if (PyArray_DIM(ids, 0) != m) Py_RETURN_FALSE;
  const npy_int64* p = (const npy_int64*)PyArray_DATA(ids);
  for (npy_intp i = 0; i < m; ++i)
    if (p[i] != (npy_int64)(intptr_t)PyList_GET_ITEM(lst, i)) Py_RETURN_FALSE;
  Py_RETURN_TRUE;
}

static PyObject* concat_ragged(PyObject* self, PyObject* args) {
  PyObject* lst;
  PyArrayObject* lens;
  (void)self;
  if (!PyArg_ParseTuple(args, "O!O!", &PyList_Type, &lst, &PyArray_Type, &lens)) return NULL;
  if (PyArray_NDIM(lens) != 1 || PyArray_TYPE(lens) != NPY_INT64 || !PyArray_ISCARRAY_RO(lens) ||
      PyArray_DIM(lens, 0) != PyList_GET_SIZE(lst)) {
    PyErr_SetString(PyExc_ValueError, "concat_ragged: need int64 lengths, one per list element");
    return NULL;
  }
  const npy_intp m = PyList_GET_SIZE(lst);
  const npy_int64* ln = (const npy_int64*)PyArray_DATA(lens);
  npy_intp total = 0;
  for (npy_intp i = 0; i < m; ++i) {
    PyObject* e = PyList_GET_ITEM(lst, i);
    if (!PyArray_Check(e)) {
      PyErr_SetString(PyExc_TypeError, "concat_ragged: element is not an ndarray");
      return NULL;
    }
    PyArrayObject* a = (PyArrayObject*)e;
    const int t = PyArray_TYPE(a);
    if (PyArray_NDIM(a) != 1 || !PyArray_ISCARRAY_RO(a) ||
        !(t == NPY_INT64 || t == NPY_INT32 || t == NPY_INT16 || t == NPY_UINT16 || t == NPY_UINT8)) {
      PyErr_SetString(PyExc_TypeError, "concat_ragged: element is not a contiguous 1-D integer array");
      return NULL;
    }
    if (ln[i] < 0 || PyArray_DIM(a, 0) < ln[i]) {
      PyErr_SetString(PyExc_ValueError, "word lists shorter than the document lengths");
      return NULL;
    }
    total += (npy_intp)ln[i];
  }
  PyObject* out = PyArray_SimpleNew(1, &total, NPY_INT32);
  if (!out) return NULL;
  int32_t* dst = (int32_t*)PyArray_DATA((PyArrayObject*)out);
  int64_t lo = INT64_MAX, hi = INT64_MIN;
  for (npy_intp i = 0; i < m; ++i) {
    PyArrayObject* a = (PyArrayObject*)PyList_GET_ITEM(lst, i);
    const npy_intp n = (npy_intp)ln[i];
    const char* src = PyArray_BYTES(a);
    switch (PyArray_TYPE(a)) {
      case NPY_INT64: {
        const int64_t* s = (const int64_t*)src;
        for (npy_intp k = 0; k < n; ++k) {
          const int64_t v = s[k];
          lo = v < lo ? v : lo;
          hi = v > hi ? v : hi;
          dst[k] = (int32_t)v;
        }
        break;
      }
      case NPY_INT32: {
        const int32_t* s = (const int32_t*)src;
        for (npy_intp k = 0; k < n; ++k) {
          lo = s[k] < lo ? s[k] : lo;
          hi = s[k] > hi ? s[k] : hi;
        }
        memcpy(dst, s, (size_t)n * sizeof(int32_t));
        break;
      }
      case NPY_INT16: {
        const int16_t* s = (const int16_t*)src;
        for (npy_intp k = 0; k < n; ++k) {
          lo = s[k] < lo ? s[k] : lo;
          hi = s[k] > hi ? s[k] : hi;
          dst[k] = s[k];
        }
        break;
      }
      case NPY_UINT16: {
        const uint16_t* s = (const uint16_t*)src;
        for (npy_intp k = 0; k < n; ++k) {
          hi = s[k] > hi ? s[k] : hi;
          lo = s[k] < lo ? s[k] : lo;
          dst[k] = s[k];
        }
        break;
      }
      default: {
        const uint8_t* s = (const uint8_t*)src;
        for (npy_intp k = 0; k < n; ++k) {
          hi = s[k] > hi ? s[k] : hi;
          lo = s[k] < lo ? s[k] : lo;
          dst[k] = s[k];
        }
        break;
      }
    }
    dst += n;
  }
  if (total == 0) lo = 0, hi = -1;
  if (lo < INT32_MIN || hi > INT32_MAX) {
    Py_DECREF(out);
    PyErr_Format(PyExc_OverflowError, "word id %lld does not fit the int32 device layout",
                 (long long)(hi > INT32_MAX ? hi : lo));
    return NULL;
  }
  return Py_BuildValue("(NLL)", out, (long long)lo, (long long)hi);
}


/* ---------------------------------------------------------------- widen */
typedef struct {
  const int32_t* src;
  int64_t* dst;
  npy_intp a, b;
} widen_job;

static void* widen_worker(void* arg) {
  widen_job* j = (widen_job*)arg;
  for (npy_intp i = j->a; i < j->b; ++i) j->dst[i] = j->src[i];
  return NULL;
}

static void unmap_capsule(PyObject* cap) {
  void* p = PyCapsule_GetPointer(cap, "wd_mmap");
  size_t* sz = (size_t*)PyCapsule_GetContext(cap);
  if (p && sz) munmap(p, *sz);
  free(sz);
}

static PyObject* widen_i32(PyObject* self, PyObject* args) {
  unsigned long long addr;
  Py_ssize_t n;
  int threads;
  (void)self;
  if (!PyArg_ParseTuple(args, "Kni", &addr, &n, &threads)) return NULL;
  if (n < 0 || (n > 0 && addr == 0)) {
    PyErr_SetString(PyExc_ValueError, "widen_i32: bad buffer");
    return NULL;
  }
  const size_t bytes = (size_t)(n > 0 ? n : 1) * sizeof(int64_t);
  const size_t huge = (size_t)2 << 20;
  const size_t len = (bytes + huge - 1) / huge * huge;
  void* mem = mmap(NULL, len, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
  if (mem == MAP_FAILED) return PyErr_NoMemory();
  madvise(mem, len, MADV_HUGEPAGE);
  int T = threads < 1 ? 1 : (threads > 64 ? 64 : threads);
  if (n < ((npy_intp)1 << 20)) T = 1;
  pthread_t th[64];
  widen_job jobs[64];
  Py_BEGIN_ALLOW_THREADS;
  for (int t = 0; t < T; ++t) {
    jobs[t].src = (const int32_t*)(uintptr_t)addr;
    jobs[t].dst = (int64_t*)mem;
    jobs[t].a = (npy_intp)((int64_t)n * t / T);
    jobs[t].b = (npy_intp)((int64_t)n * (t + 1) / T);
    if (T > 1) pthread_create(&th[t], NULL, widen_worker, &jobs[t]);
    else widen_worker(&jobs[t]);
  }
  if (T > 1)
    for (int t = 0; t < T; ++t) pthread_join(th[t], NULL);
  Py_END_ALLOW_THREADS;
  npy_intp dims[1] = {n};
  PyObject* arr = PyArray_SimpleNewFromData(1, dims, NPY_INT64, mem);
  if (!arr) {
    munmap(mem, len);
    return NULL;
  }
  size_t* szp = (size_t*)malloc(sizeof(size_t));
  if (!szp) {
    Py_DECREF(arr);
    munmap(mem, len);
    return PyErr_NoMemory();
  }
  *szp = len;
  PyObject* cap = PyCapsule_New(mem, "wd_mmap", unmap_capsule);
  if (!cap) {
    free(szp);
    Py_DECREF(arr);
    munmap(mem, len);
    return NULL;
  }
  PyCapsule_SetContext(cap, szp);
  if (PyArray_SetBaseObject((PyArrayObject*)arr, cap) < 0) {
    Py_DECREF(arr);
    return NULL;
  }
  return arr;
}

static PyMethodDef methods[] = {
    {"ragged_views", ragged_views, METH_VARARGS, "list of views z[offsets[m]:offsets[m+1]]"},
    {"list_ids", list_ids, METH_O, "int64 ids of the list's elements"},
    {"ids_equal", ids_equal, METH_VARARGS, "same list elements (by identity)"},
    {"concat_ragged", concat_ragged, METH_VARARGS, "(int32 words, min, max) of a ragged corpus"},
    {"widen_i32", widen_i32, METH_VARARGS, "fresh int64 array (huge pages) of n int32 at an address"},
    {NULL, NULL, 0, NULL}};

static struct PyModuleDef module = {PyModuleDef_HEAD_INIT, "_wdhost", "warpdraw B200 host helpers", -1, methods,
                                    NULL, NULL, NULL, NULL};

PyMODINIT_FUNC PyInit__wdhost(void) {
  import_array();
  return PyModule_Create(&module);
}
