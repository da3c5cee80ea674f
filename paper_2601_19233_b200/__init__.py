"""UniMGS single-pass anti-aliased mesh + 3DGS rasterizer, B200-native (sm_100a).

The compute path lives in libunimgs.so (csrc/, C ABI in include/unimgs.h);
``renderer`` is a ctypes binding over it, ``scenes`` the seeded synthetic
input generators, ``dist`` the camera-view sharding across GPUs.
"""
__all__ = ["scenes", "renderer", "dist", "build"]
