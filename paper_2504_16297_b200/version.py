"""Version of the drop-in API surface.

The manifest's ``engine`` block keeps the reference's name and version
(``pkg/src/trajsim/version.py:1``, ``execute.py:207``) so datasets written by
this engine compare equal to the reference's under ``manifest_core``.
"""

__version__ = "0.1.0"
ENGINE_NAME = "trajsim"
BACKEND = "ptsbe-b200"
