"""Build tools/replay/replay_ext.cpp in-tree (tools/replay/_build)."""
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
BUILD = os.path.join(HERE, "_build")


def build():
    from torch.utils.cpp_extension import load
    os.makedirs(BUILD, exist_ok=True)
    return load(name="memplan_replay_ext", sources=[os.path.join(HERE, "replay_ext.cpp")],
                build_directory=BUILD, with_cuda=True, extra_cflags=["-O3"], verbose=False)


def import_built():
    if BUILD not in sys.path:
        sys.path.insert(0, BUILD)
    import memplan_replay_ext  # noqa: E402
    return memplan_replay_ext


if __name__ == "__main__":
    build()
    print("built", BUILD)
