"""Build the oracle's native pieces (none yet beyond numpy/torch); kept for the build() contract."""


def build() -> None:
    return None
