"""Test helper: temporarily set environment switches (read by the native
library when a handle is created)."""
import contextlib
import os


@contextlib.contextmanager
def layout_env(**env):
    old = {k: os.environ.get(k) for k in env}
    os.environ.update({k: str(v) for k, v in env.items()})
    try:
        yield
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k)
            else:
                os.environ[k] = v
