/* blp_pyobj.c -- CPython extension `_pyobj`: marshalling of the reference's object
 * API (batch_solve(list[StandardFormLP]), /root/reference/pkg/src/batchlp/batch.py:134-179)
 * into the C ABI's gather entry point (blp_solve_batch_gather, include/blp.h).
 *
 * collect(lps, m, n) walks the list once under the GIL and returns, for every LP,
 * the addresses of its A, b and c data when each is a C-contiguous float64 buffer of
 * the batch shape (numpy arrays built by standard_form / the generators are), so the
 * library can copy them straight into its pinned staging ring with host threads --
 * no np.stack, no per-LP Python objects.  LPs whose arrays are anything else (lists,
 * other dtypes, strided views) are reported in `slow` for the Python side to coerce.
 * It also counts negative b entries (the batch-worst artificial count of the chunk
 * plan, batch.py:146-152) and finds the first LP whose (len(b), len(c)) differs from
 * (m, n) (HeterogeneousBatch); an A that is not an m x n float64 buffer is a slow LP.
 *
 * Returns (ptrs: bytes of int64[3][count], slow: list[int], worst_neg: int,
 *          first_hetero: int)   (-1 = none).
 * The caller keeps `lps` alive for as long as the pointers are used; the reference
 * API treats the arrays as immutable (model.py:44-45).
 */
#define PY_SSIZE_T_CLEAN
#include <Python.h>
#define NPY_NO_DEPRECATED_API NPY_1_7_API_VERSION
#include <numpy/arrayobject.h>
#include <stdint.h>
#include <string.h>

static PyObject *s_A, *s_b, *s_c;

/* Buffer of `obj` if it is a C-contiguous float64 array with `count` elements and the
 * expected ndim/shape (ndim_want 1: (d0,), 2: (d0, d1)); else NULL (no exception set). */
static const double *f64_buffer(PyObject *obj, int ndim_want, Py_ssize_t d0, Py_ssize_t d1, int *shape_ok) {
    Py_buffer v;
    *shape_ok = -1; /* unknown */
    if (PyArray_Check(obj)) {   /* numpy fast path: no buffer-protocol round trip */
        PyArrayObject *a = (PyArrayObject *)obj;
        const npy_intp *dims = PyArray_DIMS(a);
        if (PyArray_NDIM(a) != ndim_want) { *shape_ok = 0; return NULL; }
        *shape_ok = ndim_want == 1 ? (dims[0] == d0) : (dims[0] == d0 && dims[1] == d1);
        if (*shape_ok && PyArray_TYPE(a) == NPY_DOUBLE && PyArray_ISNOTSWAPPED(a) && PyArray_IS_C_CONTIGUOUS(a))
            return (const double *)PyArray_DATA(a);
        return NULL;
    }
    if (!PyObject_CheckBuffer(obj)) return NULL;
    if (PyObject_GetBuffer(obj, &v, PyBUF_RECORDS_RO) != 0) {
        PyErr_Clear();
        return NULL;
    }
    const double *p = NULL;
    const int fmt_ok = v.itemsize == 8 && v.format &&
                       (strcmp(v.format, "d") == 0 || strcmp(v.format, "<d") == 0 || strcmp(v.format, "=d") == 0);
    if (v.ndim == ndim_want) {
        *shape_ok = ndim_want == 1 ? (v.shape[0] == d0) : (v.shape[0] == d0 && v.shape[1] == d1);
    } else {
        *shape_ok = 0;
    }
    if (fmt_ok && *shape_ok == 1 && PyBuffer_IsContiguous(&v, 'C')) p = (const double *)v.buf;
    PyBuffer_Release(&v);
    return p;
}

static PyObject *collect(PyObject *self, PyObject *args) {
    PyObject *lps;
    Py_ssize_t m, n;
    (void)self;
    if (!PyArg_ParseTuple(args, "Onn", &lps, &m, &n)) return NULL;
    PyObject *seq = PySequence_Fast(lps, "lps must be a sequence");
    if (!seq) return NULL;
    const Py_ssize_t count = PySequence_Fast_GET_SIZE(seq);
    PyObject **items = PySequence_Fast_ITEMS(seq);
    PyObject *ptrs = PyBytes_FromStringAndSize(NULL, (Py_ssize_t)(3 * count * sizeof(int64_t)));
    PyObject *slow = PyList_New(0);
    if (!ptrs || !slow) goto fail;
    int64_t *P = (int64_t *)PyBytes_AS_STRING(ptrs);
    int64_t *PA = P, *Pb = P + count, *Pc = P + 2 * count;
    long worst_neg = 0;
    const double *last_pb = NULL;
    Py_ssize_t first_hetero = -1;
    for (Py_ssize_t k = 0; k < count; ++k) {
        PyObject *lp = items[k];
        PyObject *A = PyObject_GetAttr(lp, s_A);
        PyObject *b = A ? PyObject_GetAttr(lp, s_b) : NULL;
        PyObject *c = b ? PyObject_GetAttr(lp, s_c) : NULL;
        if (!c) {
            Py_XDECREF(A);
            Py_XDECREF(b);
            goto fail;
        }
        int ok_b, ok_c, ok_A;
        const double *pb = f64_buffer(b, 1, m, 0, &ok_b);
        const double *pc = f64_buffer(c, 1, n, 0, &ok_c);
        const double *pA = f64_buffer(A, 2, m, n, &ok_A);
        if (ok_b != 1 || ok_c != 1) {
            /* not a 1-D buffer of the batch length: decide with len(), the reference's lp.m / lp.n */
            const Py_ssize_t lb = PyObject_Length(b), lc = PyObject_Length(c);
            if (lb < 0 || lc < 0) {
                Py_DECREF(A); Py_DECREF(b); Py_DECREF(c);
                goto fail;
            }
            if ((lb != m || lc != n) && first_hetero < 0) first_hetero = k;
        }
        /* anything but three float64 C-contiguous buffers of the batch shape: Python coerces */
        const int slow_lp = !pA || !pb || !pc;
        if (slow_lp) {
            PyObject *ik = PyLong_FromSsize_t(k);
            if (!ik || PyList_Append(slow, ik) != 0) {
                Py_XDECREF(ik);
                Py_DECREF(A); Py_DECREF(b); Py_DECREF(c);
                goto fail;
            }
            Py_DECREF(ik);
            PA[k] = Pb[k] = Pc[k] = 0;
        } else {
            PA[k] = (int64_t)(intptr_t)pA;
            Pb[k] = (int64_t)(intptr_t)pb;
            Pc[k] = (int64_t)(intptr_t)pc;
            if (pb != last_pb) {   /* one shared b (support function): counted once */
                long neg = 0;
                for (Py_ssize_t i = 0; i < m; ++i) neg += pb[i] < 0.0;
                if (neg > worst_neg) worst_neg = neg;
                last_pb = pb;
            }
        }
        Py_DECREF(A);
        Py_DECREF(b);
        Py_DECREF(c);
    }
    Py_DECREF(seq);
    return Py_BuildValue("NNln", ptrs, slow, worst_neg, first_hetero);
fail:
    Py_XDECREF(ptrs);
    Py_XDECREF(slow);
    Py_DECREF(seq);
    return NULL;
}

static PyMethodDef methods[] = {
    {"collect", collect, METH_VARARGS, "collect(lps, m, n) -> (ptrs, slow, worst_neg, first_hetero)"},
    {NULL, NULL, 0, NULL},
};

static struct PyModuleDef module = {PyModuleDef_HEAD_INIT, "_pyobj", "StandardFormLP list marshalling", -1, methods};

PyMODINIT_FUNC PyInit__pyobj(void) {
    import_array();
    s_A = PyUnicode_InternFromString("A");
    s_b = PyUnicode_InternFromString("b");
    s_c = PyUnicode_InternFromString("c");
    return PyModule_Create(&module);
}
