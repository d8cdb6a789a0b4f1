"""B200-native ParisKV decode-time KV-cache retrieval hot path (arXiv 2602.07721).

The product is the C-ABI library libpariskv.so (include/pariskv.h, CUDA kernels for sm_100a in csrc/);
`pariskv` is its thin ctypes binding with the same entry-point names. Accessing the binding without the
built library raises ImportError (there is no CPU fallback). `build` compiles the library with nvcc."""
_API = ("Config", "Index", "append_decode_keys", "config_init", "encode_keys", "retrieve_topk", "schedule",
        "sparse_attend")


def __getattr__(name):
    if name == "pariskv" or name in _API:
        import importlib
        mod = importlib.import_module(__name__ + ".pariskv")
        return mod if name == "pariskv" else getattr(mod, name)
    raise AttributeError(name)
