"""Exception types, mirroring pkg/src/stmp/errors.py:4-24."""


class FormatError(ValueError):
    """A binary file does not match its declared layout."""


class StaleTreeError(RuntimeError):
    """A cluster tree does not belong to the dictionary it is used with (errors.py:19-20)."""
