/* Python int <-> limb conversion for the drop-in run_vector / run_ntt calls
 * (reference kernels.to_words / from_words, kernels.py:418-428, and the
 * per-element Python loops of run_vector / run_ntt, kernels.py:467-499).
 *
 * The values cross the boundary as Python ints; this CPython extension moves
 * them to and from little-endian 32-bit limbs with the interpreter's own
 * byte-array conversions, one C loop per call instead of one Python-level
 * int.to_bytes / int.from_bytes per element.  Host-side marshalling only:
 * every modular operation runs in libwidemod_b200.so on the device.
 */
#define PY_SSIZE_T_CLEAN
#include <Python.h>
#include <string.h>

#if PY_VERSION_HEX >= 0x030D0000
#define WM_AS_BYTES(v, p, n) _PyLong_AsByteArray((PyLongObject *)(v), (p), (n), 1, 0, 1)
#else
#define WM_AS_BYTES(v, p, n) _PyLong_AsByteArray((PyLongObject *)(v), (p), (n), 1, 0)
#endif

/* ints_to_limbs(values, limbs) -> bytes of len(values) * limbs * 4 */
static PyObject *ints_to_limbs(PyObject *self, PyObject *args) {
  PyObject *seq_in;
  Py_ssize_t limbs;
  if (!PyArg_ParseTuple(args, "On", &seq_in, &limbs)) return NULL;
  if (limbs < 1) {
    PyErr_SetString(PyExc_ValueError, "limbs must be >= 1");
    return NULL;
  }
  PyObject *seq = PySequence_Fast(seq_in, "expected a sequence of ints");
  if (!seq) return NULL;
  const Py_ssize_t n = PySequence_Fast_GET_SIZE(seq);
  const size_t per = (size_t)limbs * 4;
  PyObject *out = PyBytes_FromStringAndSize(NULL, (Py_ssize_t)(per * (size_t)n));
  if (!out) {
    Py_DECREF(seq);
    return NULL;
  }
  unsigned char *dst = (unsigned char *)PyBytes_AS_STRING(out);
  PyObject **items = PySequence_Fast_ITEMS(seq);
  for (Py_ssize_t i = 0; i < n; ++i) {
    PyObject *v = items[i];
    PyObject *tmp = NULL;
    if (!PyLong_Check(v)) {
      tmp = PyNumber_Index(v);
      if (!tmp) goto fail;
      v = tmp;
    }
    if (_PyLong_Sign(v) < 0) {
      Py_XDECREF(tmp);
      PyErr_SetString(PyExc_OverflowError, "negative value");
      goto fail;
    }
    if (WM_AS_BYTES(v, dst + per * (size_t)i, per) < 0) {
      Py_XDECREF(tmp);
      goto fail; /* OverflowError: does not fit in `limbs` limbs */
    }
    Py_XDECREF(tmp);
  }
  Py_DECREF(seq);
  return out;
fail:
  Py_DECREF(seq);
  Py_DECREF(out);
  return NULL;
}

/* limbs_to_ints(buffer, limbs) -> list of ints (buffer: n * limbs uint32, little-endian) */
static PyObject *limbs_to_ints(PyObject *self, PyObject *args) {
  Py_buffer buf;
  Py_ssize_t limbs;
  if (!PyArg_ParseTuple(args, "y*n", &buf, &limbs)) return NULL;
  const size_t per = (size_t)limbs * 4;
  if (limbs < 1 || buf.len % (Py_ssize_t)per) {
    PyBuffer_Release(&buf);
    PyErr_SetString(PyExc_ValueError, "buffer is not a whole number of values");
    return NULL;
  }
  const Py_ssize_t n = buf.len / (Py_ssize_t)per;
  PyObject *list = PyList_New(n);
  if (!list) {
    PyBuffer_Release(&buf);
    return NULL;
  }
  const unsigned char *src = (const unsigned char *)buf.buf;
  for (Py_ssize_t i = 0; i < n; ++i) {
    PyObject *v = _PyLong_FromByteArray(src + per * (size_t)i, per, 1, 0);
    if (!v) {
      Py_DECREF(list);
      PyBuffer_Release(&buf);
      return NULL;
    }
    PyList_SET_ITEM(list, i, v);
  }
  PyBuffer_Release(&buf);
  return list;
}

static PyMethodDef methods[] = {
    {"ints_to_limbs", ints_to_limbs, METH_VARARGS, "Python ints -> little-endian uint32 limbs (bytes)."},
    {"limbs_to_ints", limbs_to_ints, METH_VARARGS, "little-endian uint32 limbs (buffer) -> list of ints."},
    {NULL, NULL, 0, NULL}};

static struct PyModuleDef module = {PyModuleDef_HEAD_INIT, "_wmconv", NULL, -1, methods};

PyMODINIT_FUNC PyInit__wmconv(void) { return PyModule_Create(&module); }
