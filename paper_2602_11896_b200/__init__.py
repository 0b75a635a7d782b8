"""B200-native JTFS forward + gradient + metamer step (arxiv 2602.11896), via libjtfs.so.

`Plan` (jtfs.py) wraps the C ABI declared in include/jtfs.h; `dist` holds the torch.distributed
glue (batch sharding and path sharding with one all_reduce of dE/dx and the loss)."""
from .jtfs import Plan, JtfsError  # noqa: F401
