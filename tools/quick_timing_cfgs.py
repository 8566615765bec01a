"""Configs shared by the scratch timing tools (BASELINE.json configs)."""
CFGS = {
    1: dict(shape=(256, 256), ratio=0.25, kind="uniform-random", patch=(8, 8), k=64, epochs=10),
    3: dict(shape=(512, 512), ratio=0.25, kind="line-hop", patch=(8, 8), k=256, epochs=2),
    2: dict(shape=(1024, 1024), ratio=0.10, kind="uniform-random", patch=(10, 10), k=256, epochs=3),
    4: dict(shape=(256, 256, 128), ratio=0.20, kind="uniform-random", patch=(8, 8, 4), k=512, epochs=2),
    5: dict(shape=(4096, 4096), ratio=0.10, kind="uniform-random", patch=(8, 8), k=256, epochs=2),
}
